"""Word-size model of a redundant representation for the FULL modulus class (q >= 2^(w-1),
the 128-bit class q >= 2^127 scaled down to w-bit words): values kept in [0, 2^w) instead of
[0, q) between butterfly stages.  Exhaustive over every odd q in
(2^(w-1), 2^w) and every operand pair, w = 8 and 10:

  mont  : T in [0, 2q) -> T - q when bit w is set           (always < 2^w, always valid)
  add1  : s = u + t, one carry-masked -q                     (NOT closed: s - q >= 2^w happens)
  add2  : ... and a second carry-masked -q                   (closed, but two corrections)
  sub2  : d = u - t, up to two borrow-masked +q              (closed)

Result printed per rule: pairs checked, failures.  The canonical butterfly needs one
compare-and-select per add / sub / Montgomery output ("FULL class"); the
redundant one needs the same Montgomery correction and TWO masked corrections per add, so
it executes more ALU operations, not fewer."""
import sys


def check(w):
    W = 1 << w
    res = {"mont": [0, 0], "add1": [0, 0], "add2": [0, 0], "sub2": [0, 0]}
    for q in range(W // 2 + 1, W, 2):
        for T in range(0, 2 * q):                           # Montgomery output range
            r = T - q if T >= W else T
            res["mont"][0] += 1
            res["mont"][1] += not (0 <= r < W and r % q == T % q)
        for u in range(W):
            for t in range(W):
                s = u + t
                a1 = s - q if s >= W else s
                res["add1"][0] += 1
                res["add1"][1] += not (0 <= a1 < W)
                a2 = a1 - q if a1 >= W else a1
                res["add2"][0] += 1
                res["add2"][1] += not (0 <= a2 < W and a2 % q == s % q)
                d = u - t
                d1 = d + q if d < 0 else d
                d2 = d1 + q if d1 < 0 else d1
                res["sub2"][0] += 1
                res["sub2"][1] += not (0 <= d2 < W and d2 % q == (u - t) % q)
    return res


if __name__ == "__main__":
    for w in (8, 10) if len(sys.argv) < 2 else [int(v) for v in sys.argv[1:]]:
        for k, (n, f) in check(w).items():
            print(f"w={w} {k:5s} checked {n:9d} failures {f}")
