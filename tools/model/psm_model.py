"""Word-level model of csrc/psm128.cuh (pseudo-Mersenne class, q = 2^b - c, Q = q 2^s =
2^128 - C with C < 2^32): every instruction of psm_add / psm_sub / psm_mul / psm_canon on
32-bit words with an explicit carry flag, asserting each dropped carry is zero and each
result against Python integers.  A development model of the kernel arithmetic (run by
tests/test_psm_model.py), not the oracle."""
M32 = 0xFFFFFFFF
R = 1 << 128


class Flag:
    """the CC.CF carry / borrow flag of the PTX .cc instructions"""

    def __init__(self):
        self.c = 0

    def add(self, x, y, cin=False, cout=True):
        t = x + y + (self.c if cin else 0)
        if cout:
            self.c = t >> 32
        else:
            assert t >> 32 == 0, "dropped carry"
        return t & M32

    def sub(self, x, y, bin_=False, bout=True):
        t = x - y - (self.c if bin_ else 0)
        if bout:
            self.c = 1 if t < 0 else 0
        else:
            assert t >= 0, "dropped borrow"
        return t & M32

    def mad_lo(self, a, b, c, cin=False, cout=True):
        return self.add((a * b) & M32, c, cin, cout)

    def mad_hi(self, a, b, c, cin=False, cout=True):
        return self.add((a * b) >> 32, c, cin, cout)


def words(x, n=4):
    return [(x >> (32 * i)) & M32 for i in range(n)]


def val(w):
    return sum(x << (32 * i) for i, x in enumerate(w))


def params(q):
    b = q.bit_length()
    s = 128 - b
    Q = q << s
    assert Q >> 32 == (1 << 96) - 1, "not in the class"
    C = (-((q & M32) << s)) & M32
    assert R - Q == C and C >= 1
    assert C != M32, "C = 2^32 - 1 is excluded (psm_mul's l4 + 1)"
    return s, C


def psm_add(a, b, C):
    A, B = words(a), words(b)
    f = Flag()
    s = [f.add(A[0], B[0])] + [f.add(A[i], B[i], True) for i in (1, 2, 3)]
    k = f.c
    s[0] = f.add(s[0], C if k else 0)
    for i in (1, 2, 3):
        s[i] = f.add(s[i], 0, True)
    k = f.c
    if k:
        assert s[1] == s[2] == s[3] == 0 and s[0] < C
    s[0] = f.add(s[0], C if k else 0)
    s[1] = f.add(s[1], 0, True, cout=False)
    return val(s)


def psm_sub(a, b, C):
    A, B = words(a), words(b)
    f = Flag()
    d = [f.sub(A[0], B[0])] + [f.sub(A[i], B[i], True) for i in (1, 2, 3)]
    bw = f.c
    d[0] = f.sub(d[0], C if bw else 0)
    for i in (1, 2, 3):
        d[i] = f.sub(d[i], 0, True)
    bw = f.c
    if bw:
        assert d[1] == d[2] == d[3] == M32
    d[0] = f.sub(d[0], C if bw else 0)
    d[1] = f.sub(d[1], 0, True, bout=False)
    return val(d)


def psm_mul(a, b, C):
    A, B = words(a), words(b)
    f = Flag()
    e = [0] * 8
    for pos, (i, j) in ((0, (0, 0)), (2, (0, 2)), (4, (1, 3)), (6, (3, 3))):
        p = A[i] * B[j]
        e[pos], e[pos + 1] = p & M32, p >> 32
    for (i1, j1), (i2, j2) in (((1, 1), (2, 2)), ((2, 0), (3, 1))):
        e[2] = f.mad_lo(A[i1], B[j1], e[2])
        e[3] = f.mad_hi(A[i1], B[j1], e[3], True)
        e[4] = f.mad_lo(A[i2], B[j2], e[4], True)
        e[5] = f.mad_hi(A[i2], B[j2], e[5], True)
        e[6] = f.add(e[6], 0, True)
        e[7] = f.add(e[7], 0, True, cout=False)
    o = [0] * 7
    for pos, (i, j) in ((0, (0, 1)), (2, (0, 3)), (4, (2, 3))):
        p = A[i] * B[j]
        o[pos], o[pos + 1] = p & M32, p >> 32
    o[0] = f.mad_lo(A[1], B[0], o[0])
    o[1] = f.mad_hi(A[1], B[0], o[1], True)
    o[2] = f.mad_lo(A[1], B[2], o[2], True)
    o[3] = f.mad_hi(A[1], B[2], o[3], True)
    o[4] = f.mad_lo(A[3], B[2], o[4], True)
    o[5] = f.mad_hi(A[3], B[2], o[5], True)
    o[6] = f.add(0, 0, True, cout=False)
    for (i, j) in ((2, 1), (3, 0)):
        o[2] = f.mad_lo(A[i], B[j], o[2])
        o[3] = f.mad_hi(A[i], B[j], o[3], True)
        o[4] = f.add(o[4], 0, True)
        o[5] = f.add(o[5], 0, True)
        o[6] = f.add(o[6], 0, True, cout=False)
    e[1] = f.add(e[1], o[0])
    for i in range(2, 7):
        e[i] = f.add(e[i], o[i - 1], True)
    e[7] = f.add(e[7], o[6], True, cout=False)
    assert val(e) == a * b
    h = e[4:8]
    e[0] = f.mad_lo(h[0], C, e[0])
    e[1] = f.mad_hi(h[0], C, e[1], True)
    e[2] = f.mad_lo(h[2], C, e[2], True)
    e[3] = f.mad_hi(h[2], C, e[3], True)
    l4 = f.add(0, 0, True, cout=False)
    e[1] = f.mad_lo(h[1], C, e[1])
    e[2] = f.mad_hi(h[1], C, e[2], True)
    e[3] = f.mad_lo(h[3], C, e[3], True)
    l4 = f.mad_hi(h[3], C, l4, True, cout=False)
    assert val(e[:4]) + (l4 << 128) == (a * b) % R + ((a * b) >> 128) * C
    m = l4 + 1
    assert m <= M32 and l4 <= C
    e[0] = f.mad_lo(m, C, e[0])
    e[1] = f.mad_hi(m, C, e[1], True)
    e[2] = f.add(e[2], 0, True)
    e[3] = f.add(e[3], 0, True)
    k = f.c
    e[0] = f.sub(e[0], 0 if k else C)
    e[1] = f.sub(e[1], 0, True)
    e[2] = f.sub(e[2], 0, True)
    e[3] = f.sub(e[3], 0, True, bout=False)
    return val(e[:4])


def psm_add1(a, t, C):
    """t < Q: a single fold"""
    A, B = words(a), words(t)
    f = Flag()
    s = [f.add(A[0], B[0])] + [f.add(A[i], B[i], True) for i in (1, 2, 3)]
    k = f.c
    s[0] = f.add(s[0], C if k else 0)
    s[1] = f.add(s[1], 0, True)
    s[2] = f.add(s[2], 0, True)
    s[3] = f.add(s[3], 0, True, cout=False)
    return val(s)


def psm_sub1(a, t, C):
    A, B = words(a), words(t)
    f = Flag()
    d = [f.sub(A[0], B[0])] + [f.sub(A[i], B[i], True) for i in (1, 2, 3)]
    bw = f.c
    d[0] = f.sub(d[0], C if bw else 0)
    d[1] = f.sub(d[1], 0, True)
    d[2] = f.sub(d[2], 0, True)
    d[3] = f.sub(d[3], 0, True, bout=False)
    return val(d)


def psm_canon(v, q, s, C):
    V = words(v)
    vh = (V[3] >> (32 - s)) if s else 0
    top = V[3] & (M32 >> s)
    add = vh * (C >> s)
    assert add <= M32
    f = Flag()
    r = [f.add(V[0], add), f.add(V[1], 0, True), f.add(V[2], 0, True), f.add(top, 0, True, cout=False)]
    x = val(r)
    assert x < 2 * q
    return x - q if x >= q else x


def check(q, a, b):
    """a, b: any 128-bit values; the product takes b mod q (a twiddle is canonical), and the
    butterfly (a + a w, a - a w forms: u = b, v = a, w = b mod q) takes the single-fold add / sub"""
    s, C = params(q)
    Q = q << s
    for fn, ref in ((psm_add, a + b), (psm_sub, a - b)):
        r = fn(a, b, C)
        assert 0 <= r < R and (r - ref) % Q == 0, (fn.__name__, hex(q), hex(a), hex(b))
        assert psm_canon(r, q, s, C) == ref % q, ("canon", fn.__name__, hex(q), hex(a), hex(b))
    for w in {b % q, q - 1, 1, 0}:
        t = psm_mul(a, w, C)
        assert 0 <= t < Q and (t - a * w) % Q == 0, ("mul", hex(q), hex(a), hex(w))
        assert psm_canon(t, q, s, C) == (a * w) % q
        for u in (a, b, R - 1, 0):
            for fn, ref in ((psm_add1, u + t), (psm_sub1, u - t)):
                r = fn(u, t, C)
                assert 0 <= r < R and (r - ref) % Q == 0, (fn.__name__, hex(q), hex(u), hex(t))


def edge_values(q):
    s, C = params(q)
    Q = q << s
    out = {0, 1, 2, C - 1, C, C + 1, q - 1, q, q + 1, Q - 1, Q, Q + 1, R - 1, R - 2, R - C, R - C - 1, R - C + 1,
           R - 2 * C, (1 << 64) - 1, 1 << 64, (1 << 96) - 1, R - (1 << 96), R - (1 << 64), R - (1 << 32), (1 << 127),
           (1 << 127) - 1, R - C // 2, R - C // 2 - 1}
    return sorted(x for x in out if 0 <= x < R)
