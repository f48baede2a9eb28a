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
    print(f"W={W}: {cnt} products, all carries accounted for, T < 2q, T = a b R^-1 mod q")


if __name__ == "__main__":
    main()
