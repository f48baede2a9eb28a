"""Word-level model of the even/odd alternating Montgomery product for W 32-bit words
(arith128.cuh mont_core for W = 4, arith256.cuh mont_mul256 for W = 8).  Every PTX
carry-chain op is emulated with an explicit carry flag; every place the PTX drops a carry
(a chain ending without .cc, an addend assumed not to overflow) is asserted.  Checks
T = a b R^-1 (mod q) and T < 2q against Python integers on random and edge operands.

    python tools/model/mont_eo_model_w.py 8 20000

Development model of the kernel arithmetic (not the oracle, not product code)."""
import random
import sys

M32 = (1 << 32) - 1


class Chain:
    """PTX carry flag semantics for one asm block"""

    def __init__(self):
        self.cf = 0

    def add_cc(self, a, b):
        s = a + b
        self.cf = s >> 32
        return s & M32

    def addc_cc(self, a, b):
        s = a + b + self.cf
        self.cf = s >> 32
        return s & M32

    def addc(self, a, b):               # carry out must be zero
        s = a + b + self.cf
        assert s >> 32 == 0, "dropped carry (addc)"
        return s

    def mad_pair(self, lo, hi, x, y, carry_in, carry_out=True):
        """(lo, hi) += x*y (+CF); mad.lo.cc + madc.hi(.cc)"""
        p = x * y
        s = lo + (p & M32) + (self.cf if carry_in else 0)
        t = hi + (p >> 32) + (s >> 32)
        if not carry_out:
            assert t >> 32 == 0, "dropped carry (madc.hi)"
        self.cf = t >> 32
        return s & M32, t & M32


def words(v, W):
    return [(v >> (32 * i)) & M32 for i in range(W)]


def val(w):
    return sum(x << (32 * i) for i, x in enumerate(w))


def mont_eo(a, b, q, qinv0, W):
    """returns T (W+1 words) exactly as the device code computes it"""
    H = W // 2
    # digit 0: X = a_even b0, Y = a_odd b0 (fresh products, pair aligned)
    X = [0] * (W + 1)
    Y = [0] * (W + 1)
    for k in range(H):
        p = a[2 * k] * b[0]
        X[2 * k], X[2 * k + 1] = p & M32, p >> 32
        p = a[2 * k + 1] * b[0]
        Y[2 * k], Y[2 * k + 1] = p & M32, p >> 32
    m = (X[0] * qinv0) & M32
    c = Chain()
    for k in range(H):
        X[2 * k], X[2 * k + 1] = c.mad_pair(X[2 * k], X[2 * k + 1], m, q[2 * k], k > 0)
    X[W] = c.addc(0, 0)
    c = Chain()
    for k in range(H):
        Y[2 * k], Y[2 * k + 1] = c.mad_pair(Y[2 * k], Y[2 * k + 1], m, q[2 * k + 1], k > 0)
    Y[W] = c.addc(0, 0)
    assert X[0] == 0
    for i in range(1, W):
        Xn = Y[:]                               # X' := Y (in place) with Y0 += X1
        Yn = [0] * (W + 1)
        c = Chain()
        Xn[0] = c.add_cc(Y[0], X[1])
        # Y' = X / 2^64 + carry + a_odd b_i: addends (X2,X3) .. (X_W, 0); no carry out
        for k in range(H):
            lo = X[2 * k + 2] if 2 * k + 2 <= W else 0
            hi = X[2 * k + 3] if 2 * k + 3 <= W else 0
            Yn[2 * k], Yn[2 * k + 1] = c.mad_pair(lo, hi, a[2 * k + 1], b[i], True, carry_out=(k < H - 1))
        # X' += a_even b_i, carry -> X'_W = Y_W + CF
        c = Chain()
        for k in range(H):
            Xn[2 * k], Xn[2 * k + 1] = c.mad_pair(Xn[2 * k], Xn[2 * k + 1], a[2 * k], b[i], k > 0)
        Xn[W] = c.addc(Y[W], 0)
        m = (Xn[0] * qinv0) & M32
        c = Chain()
        for k in range(H):
            Xn[2 * k], Xn[2 * k + 1] = c.mad_pair(Xn[2 * k], Xn[2 * k + 1], m, q[2 * k], k > 0)
        Xn[W] = c.addc(Xn[W], 0)
        c = Chain()
        for k in range(H):
            Yn[2 * k], Yn[2 * k + 1] = c.mad_pair(Yn[2 * k], Yn[2 * k + 1], m, q[2 * k + 1], k > 0)
        Yn[W] = c.addc(0, 0)
        assert Xn[0] == 0
        X, Y = Xn, Yn
    # T = Y + X / 2^32
    c = Chain()
    T = [0] * (W + 1)
    T[0] = c.add_cc(Y[0], X[1])
    for k in range(1, W):
        T[k] = c.addc_cc(Y[k], X[k + 1])
    T[W] = c.addc(Y[W], 0)
    return T


def check(W, q, a, b):
    qinv0 = (-pow(q, -1, 1 << 32)) & M32
    T = mont_eo(words(a, W), words(b, W), words(q, W), qinv0, W)
    t = val(T)
    R = 1 << (32 * W)
    assert t < 2 * q, "T >= 2q"
    assert (t * R - a * b) % q == 0, "not a b R^-1"


def check_lazy(W, q, rng, n):
    """Lazy class (q < R/4, values in [0, 4q) between stages; ntt256.cu, arith256_gen.cuh):
    mont_mul*_lazy on a < 4q drops T's word W, so T[W] must be 0 and T < 2q; the Harvey
    butterfly u' = u mod 2q (reduce_c with c = 2q), t = lazy(v, w), (u' + t, u' - t + 2q) must
    stay in [0, 4q) < 2^NB (add_nored / sub_add_nored drop their carries) and be congruent
    to (u + v w, u - v w) mod q (Montgomery twiddles: w = w_true R mod q)."""
    R = 1 << (32 * W)
    assert 4 * q < R
    qinv0 = (-pow(q, -1, 1 << 32)) & M32
    edge = [0, 1, q - 1, q, 2 * q - 1, 2 * q, 3 * q, 4 * q - 1]
    pairs = [(a, b) for a in edge for b in (0, 1, q - 1)] + \
            [(rng.randrange(4 * q), rng.randrange(q)) for _ in range(n)]
    for a, b in pairs:
        T = mont_eo(words(a, W), words(b, W), words(q, W), qinv0, W)
        assert T[W] == 0, "lazy: word W not zero"
        t = val(T)
        assert t < 2 * q and (t * R - a * b) % q == 0
    for _ in range(n):
        u, v, w = rng.randrange(4 * q), rng.randrange(4 * q), rng.randrange(q)
        up = u - 2 * q if u >= 2 * q else u                       # reduce_c(u, 2q)
        t = val(mont_eo(words(v, W), words(w, W), words(q, W), qinv0, W))
        x0, x1 = up + t, up + 2 * q - t
        assert 0 <= x0 < 4 * q and 0 < x1 < 4 * q and x0 < R and x1 < R
        wt = w * pow(R, -1, q) % q
        assert (x0 - (u + v * wt)) % q == 0 and (x1 - (u - v * wt)) % q == 0
    return len(pairs) + n


def main():
    W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
    bits = 32 * W
    rng = random.Random(W)
    moduli = [(1 << bits) - 1, (1 << bits) - 189, (1 << (bits - 1)) + 1, (3 << (bits - 2)) + 1,
              rng.randrange(1 << (bits - 1), 1 << bits) | 1, (1 << (bits - 64)) + 1, 65537]
    cnt = 0
    for q in moduli:
        edge = [0, 1, q - 1, q - 2, q // 2, M32, 1 << 32, (1 << bits) - 1, (1 << (bits - 1)) - 1]
        for a in edge:
            for b in edge:
                if b < q:
                    check(W, q, a % (1 << bits), b)
                    cnt += 1
        for _ in range(n // len(moduli)):
            a = rng.randrange(1 << bits)
            if rng.random() < 0.3:
                a = (1 << bits) - 1 - rng.randrange(1 << 40)
            check(W, q, a, rng.randrange(q))
            cnt += 1
    lz = 0
    for q in [(1 << (bits - 2)) - 57 | 1, rng.randrange(1 << (bits - 3), 1 << (bits - 2)) | 1, (1 << (bits - 64)) + 1, 65537]:
        lz += check_lazy(W, q, rng, max(1, n // 8))
    print(f"W={W}: {cnt} products, all carries accounted for, T < 2q, T = a b R^-1 mod q; "
          f"lazy class (q < R/4): {lz} products / butterflies, word W zero, results in [0, 4q)")


if __name__ == "__main__":
    main()
