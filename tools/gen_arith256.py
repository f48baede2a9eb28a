"""Generate paper_2509_12494_b200/csrc/arith256_gen.cuh: 8-word (256-bit) and 6-word (192-bit)
modular arithmetic for sm_100a as inline-PTX carry chains.  The Montgomery
product is the even/odd alternating CIOS of arith128.cuh generalised to W words; its carry
structure is checked word by word by tools/model/mont_eo_model_w.py (W = 8 and W = 6).

    python tools/gen_arith256.py        (rewrites the header; it is committed)
"""
import os

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2509_12494_b200", "csrc",
                   "arith256_gen.cuh")


def asm_block(lines, outs, ins):
    """lines use {name} placeholders for operands; outs/ins: lists of (constraint, expr, name)"""
    idx = {}
    for i, (_, _, name) in enumerate(outs + ins):
        idx[name] = f"%{i}"
    def one(ln):
        if ln == "{":
            return '        "{\\n\\t"'
        if ln == "}":
            return '        "}"'
        return f'        "{ln.format(**idx)};\\n\\t"'
    body = "\n".join(one(ln) for ln in lines)
    o = ", ".join(f'"{c}"({e})' for c, e, _ in outs)
    i = ", ".join(f'"{c}"({e})' for c, e, _ in ins)
    return f"    asm({body.rstrip()}\n        : {o}\n        : {i});\n"


def gen_mont(W, lazy=False):
    H = W // 2
    NB = 32 * W
    sfx = "_lazy" if lazy else ""
    s = []
    if lazy:
        s.append(f"// Lazy Montgomery product (q < 2^{NB - 2}): T = a b 2^-{NB} + {{0, q}} in [0, 2q), no final subtraction.\n"
                 f"// T = (a b + m q) / R < q (a / R) + q < 2q for any a < R; 2q < 2^{NB - 1}, so T's word {W} is zero\n"
                 f"// (tools/model/mont_eo_model_w.py checks both on a < 4q).  Same digit loop as mont_mul{NB}.\n")
    s.append(("" if lazy else f"// Montgomery product a b 2^-{NB} mod q, canonical result (a < 2^{NB}, b < q, q odd < 2^{NB}).\n") +
             "// Even/odd alternating CIOS over 32-bit digits of b: 2^32 T_i = X + 2^32 Y, X holding the\n"
             "// products at even word positions, Y at odd ones (register-pair aligned); after a digit\n"
             "// X_0 = 0 and the shift is a change of roles (X' = Y + X_1, Y' = X / 2^64 + ...).  Per\n"
             f"// digit {2 * W} IMAD.WIDE + 1 IMAD; {2 * W * W} + {W} word products in all.\n")
    s.append(f"__device__ __forceinline__ void mont_mul{NB}{sfx}(const uint32_t a[{W}], const uint32_t b[{W}], const uint32_t q[{W}],\n"
             f"                                            uint32_t qinv0, uint32_t r[{W}]) {{\n")
    s.append(f"    uint32_t x[{W + 1}], y[{W + 1}], n[{W + 1}], m;\n")
    # digit 0
    lines, outs, ins = [], [], []
    for k in range(H):
        lines += [f"mul.lo.u32 {{x{2*k}}}, {{a{2*k}}}, {{b0}}", f"mul.hi.u32 {{x{2*k+1}}}, {{a{2*k}}}, {{b0}}",
                  f"mul.lo.u32 {{y{2*k}}}, {{a{2*k+1}}}, {{b0}}", f"mul.hi.u32 {{y{2*k+1}}}, {{a{2*k+1}}}, {{b0}}"]
    outs = [("=r", f"x[{i}]", f"x{i}") for i in range(W)] + [("=r", f"y[{i}]", f"y{i}") for i in range(W)]
    ins = [("r", f"a[{i}]", f"a{i}") for i in range(W)] + [("r", "b[0]", "b0")]
    s.append(asm_block(lines, outs, ins))
    s.append("    m = x[0] * qinv0;\n")

    def red_chain(acc, parity, fresh_top):
        lines = []
        for k in range(H):
            op_lo = "mad.lo.cc.u32" if k == 0 else "madc.lo.cc.u32"
            lines += [f"{op_lo} {{{acc}{2*k}}}, {{m}}, {{q{2*k+parity}}}, {{{acc}{2*k}}}",
                      f"madc.hi.cc.u32 {{{acc}{2*k+1}}}, {{m}}, {{q{2*k+parity}}}, {{{acc}{2*k+1}}}"]
        lines.append(f"addc.u32 {{{acc}{W}}}, 0, 0" if fresh_top else f"addc.u32 {{{acc}{W}}}, {{{acc}{W}}}, 0")
        outs = [("+r", f"{acc}[{i}]", f"{acc}{i}") for i in range(W)] + [("=r" if fresh_top else "+r", f"{acc}[{W}]", f"{acc}{W}")]
        ins = [("r", "m", "m")] + [("r", f"q[{2*k+parity}]", f"q{2*k+parity}") for k in range(H)]
        return asm_block(lines, outs, ins)

    s.append(red_chain("x", 0, True))
    s.append(red_chain("y", 1, True))
    s.append(f"#pragma unroll\n    for (int i = 1; i < {W}; i++) {{\n")
    # block A: y (becomes X') in place, n = Y'
    lines = ["add.cc.u32 {y0}, {y0}, {x1}"]
    for k in range(H):
        lo = f"{{x{2*k+2}}}"
        hi = f"{{x{2*k+3}}}" if 2 * k + 3 <= W else "0"
        last = k == H - 1
        lines += [f"madc.lo.cc.u32 {{n{2*k}}}, {{a{2*k+1}}}, {{bi}}, {lo}",
                  f"madc.hi{'' if last else '.cc'}.u32 {{n{2*k+1}}}, {{a{2*k+1}}}, {{bi}}, {hi}"]
    for k in range(H):
        op_lo = "mad.lo.cc.u32" if k == 0 else "madc.lo.cc.u32"
        lines += [f"{op_lo} {{y{2*k}}}, {{a{2*k}}}, {{bi}}, {{y{2*k}}}",
                  f"madc.hi.cc.u32 {{y{2*k+1}}}, {{a{2*k}}}, {{bi}}, {{y{2*k+1}}}"]
    lines.append(f"addc.u32 {{y{W}}}, {{y{W}}}, 0")
    outs = [("+r", f"y[{i}]", f"y{i}") for i in range(W + 1)] + [("=&r", f"n[{i}]", f"n{i}") for i in range(W)]
    ins = [("r", f"x[{i}]", f"x{i}") for i in range(1, W + 1)] + [("r", f"a[{i}]", f"a{i}") for i in range(W)] + \
          [("r", "b[i]", "bi")]
    s.append("    " + asm_block(lines, outs, ins).replace("\n    ", "\n        ").lstrip())
    s.append("        m = y[0] * qinv0;\n")
    s.append("    " + red_chain("y", 0, False).replace("\n    ", "\n        ").lstrip())
    s.append("    " + red_chain("n", 1, True).replace("\n    ", "\n        ").lstrip())
    s.append(f"#pragma unroll\n        for (int k = 0; k < {W + 1}; k++) {{ x[k] = y[k]; y[k] = n[k]; }}\n    }}\n")
    if lazy:   # final: T = Y + X / 2^32 in W words (T < 2q < 2^(NB-1): no carry out)
        lines = ["add.cc.u32 {r0}, {y0}, {x1}"]
        for k in range(1, W - 1):
            lines.append(f"addc.cc.u32 {{r{k}}}, {{y{k}}}, {{x{k+1}}}")
        lines.append(f"addc.u32 {{r{W-1}}}, {{y{W-1}}}, {{x{W}}}")
        outs = [("=r", f"r[{i}]", f"r{i}") for i in range(W)]
        ins = [("r", f"y[{i}]", f"y{i}") for i in range(W)] + [("r", f"x[{i}]", f"x{i}") for i in range(1, W + 1)]
        s.append(asm_block(lines, outs, ins))
        s.append("}\n\n")
        return "".join(s)
    # final: T = Y + X / 2^32, then T - q if T >= q (T < 2q, NB + 1 bits)
    lines = ["add.cc.u32 t0, {y0}, {x1}"]
    for k in range(1, W):
        lines.append(f"addc.cc.u32 t{k}, {{y{k}}}, {{x{k+1}}}")
    lines.append(f"addc.u32 t{W}, {{y{W}}}, 0")
    lines.append("sub.cc.u32 d0, t0, {q0}")
    for k in range(1, W):
        lines.append(f"subc.cc.u32 d{k}, t{k}, {{q{k}}}")
    lines += [f"subc.u32 bw, t{W}, 0", "not.b32 nb, bw"]
    for k in range(W):
        # bw == 0: T >= q -> d; bw == ~0: T < q -> t   (r = (t & bw) | (d & ~bw))
        lines += [f"and.b32 t{k}, t{k}, bw", f"and.b32 d{k}, d{k}, nb", f"or.b32 {{r{k}}}, t{k}, d{k}"]
    regs = ", ".join([f"t{k}" for k in range(W + 1)] + [f"d{k}" for k in range(W)] + ["bw", "nb"])
    lines = ["{", f".reg .u32 {regs}"] + lines + ["}"]
    outs = [("=r", f"r[{i}]", f"r{i}") for i in range(W)]
    ins = [("r", f"y[{i}]", f"y{i}") for i in range(W + 1)] + [("r", f"x[{i}]", f"x{i}") for i in range(1, W + 1)] + \
          [("r", f"q[{i}]", f"q{i}") for i in range(W)]
    s.append(asm_block(lines, outs, ins))
    s.append("}\n\n")
    return "".join(s)


def gen_addsub(W):
    NB = 32 * W
    s = []
    # add: (NB+1)-bit sum, subtract q, select
    regs = ", ".join([f"s{k}" for k in range(W + 1)] + [f"d{k}" for k in range(W)] + ["bw", "nb"])
    lines = ["{", f".reg .u32 {regs}",
             "add.cc.u32 s0, {a0}, {b0}"] + [f"addc.cc.u32 s{k}, {{a{k}}}, {{b{k}}}" for k in range(1, W)] + \
            [f"addc.u32 s{W}, 0, 0", "sub.cc.u32 d0, s0, {q0}"] + [f"subc.cc.u32 d{k}, s{k}, {{q{k}}}" for k in range(1, W)] + \
            [f"subc.u32 bw, s{W}, 0", "not.b32 nb, bw"]
    for k in range(W):
        lines += [f"and.b32 s{k}, s{k}, bw", f"and.b32 d{k}, d{k}, nb", f"or.b32 {{r{k}}}, s{k}, d{k}"]
    lines.append("}")
    outs = [("=r", f"r[{i}]", f"r{i}") for i in range(W)]
    ins = [("r", f"a[{i}]", f"a{i}") for i in range(W)] + [("r", f"b[{i}]", f"b{i}") for i in range(W)] + \
          [("r", f"q[{i}]", f"q{i}") for i in range(W)]
    blk = asm_block(lines, outs, ins)
    s.append(f"// r = a + b mod q (Eq. saddmod, PAPER.md:184-192, {NB + 1}-bit sum); a, b < q\n")
    s.append(f"__device__ __forceinline__ void add_mod{NB}(const uint32_t a[{W}], const uint32_t b[{W}], const uint32_t q[{W}],\n"
             f"                                           uint32_t r[{W}]) {{\n" + blk + "}\n\n")
    # sub: borrow chain, + (q & mask)
    regs = ", ".join([f"d{k}" for k in range(W)] + ["bw"] + [f"m{k}" for k in range(W)])
    lines = ["{", f".reg .u32 {regs}",
             "sub.cc.u32 d0, {a0}, {b0}"] + [f"subc.cc.u32 d{k}, {{a{k}}}, {{b{k}}}" for k in range(1, W)] + \
            ["subc.u32 bw, 0, 0"] + [f"and.b32 m{k}, {{q{k}}}, bw" for k in range(W)] + \
            ["add.cc.u32 {r0}, d0, m0"] + [f"addc.cc.u32 {{r{k}}}, d{k}, m{k}" for k in range(1, W - 1)] + \
            [f"addc.u32 {{r{W-1}}}, d{W-1}, m{W-1}", "}"]
    blk = asm_block(lines, outs, ins)
    s.append("// r = a - b mod q (Eq. ssubmod, PAPER.md:193-201)\n")
    s.append(f"__device__ __forceinline__ void sub_mod{NB}(const uint32_t a[{W}], const uint32_t b[{W}], const uint32_t q[{W}],\n"
             f"                                           uint32_t r[{W}]) {{\n" + blk + "}\n\n")
    return "".join(s)


def gen_lazy(W):
    """Harvey-butterfly helpers for the lazy class (q < 2^(NB-2), values in [0, 4q))"""
    NB = 32 * W
    s = []
    outs = [("=r", f"r[{i}]", f"r{i}") for i in range(W)]
    # r = a + b, no reduction (caller: a + b < 2^NB)
    lines = ["add.cc.u32 {r0}, {a0}, {b0}"] + [f"addc.cc.u32 {{r{k}}}, {{a{k}}}, {{b{k}}}" for k in range(1, W - 1)] + \
            [f"addc.u32 {{r{W-1}}}, {{a{W-1}}}, {{b{W-1}}}"]
    ins = [("r", f"a[{i}]", f"a{i}") for i in range(W)] + [("r", f"b[{i}]", f"b{i}") for i in range(W)]
    s.append(f"// r = a + b without reduction (lazy class: a < 2q, b < 2q, r < 4q < 2^{NB})\n")
    s.append(f"__device__ __forceinline__ void add_nored{NB}(const uint32_t a[{W}], const uint32_t b[{W}], uint32_t r[{W}]) {{\n"
             + asm_block(lines, outs, ins) + "}\n\n")
    # r = a + c - b  (c = 2q; a < 2q, b < 2q: r in (0, 4q))
    regs = ", ".join(f"s{k}" for k in range(W))
    lines = ["{", f".reg .u32 {regs}", "add.cc.u32 s0, {a0}, {c0}"] + \
            [f"addc.cc.u32 s{k}, {{a{k}}}, {{c{k}}}" for k in range(1, W - 1)] + [f"addc.u32 s{W-1}, {{a{W-1}}}, {{c{W-1}}}"] + \
            ["sub.cc.u32 {r0}, s0, {b0}"] + [f"subc.cc.u32 {{r{k}}}, s{k}, {{b{k}}}" for k in range(1, W - 1)] + \
            [f"subc.u32 {{r{W-1}}}, s{W-1}, {{b{W-1}}}", "}"]
    ins = [("r", f"a[{i}]", f"a{i}") for i in range(W)] + [("r", f"b[{i}]", f"b{i}") for i in range(W)] + \
          [("r", f"c[{i}]", f"c{i}") for i in range(W)]
    s.append(f"// r = a - b + c without reduction (lazy class, c = 2q: a, b < 2q, r in (0, 4q))\n")
    s.append(f"__device__ __forceinline__ void sub_add_nored{NB}(const uint32_t a[{W}], const uint32_t b[{W}], const uint32_t c[{W}],\n"
             f"                                                 uint32_t r[{W}]) {{\n" + asm_block(lines, outs, ins) + "}\n\n")
    # r = a mod c for a < 2c (c = 2q or q): d = a - c; r = d + (c & borrow)
    regs = ", ".join([f"d{k}" for k in range(W)] + ["bw"] + [f"m{k}" for k in range(W)])
    lines = ["{", f".reg .u32 {regs}", "sub.cc.u32 d0, {a0}, {c0}"] + \
            [f"subc.cc.u32 d{k}, {{a{k}}}, {{c{k}}}" for k in range(1, W)] + ["subc.u32 bw, 0, 0"] + \
            [f"and.b32 m{k}, {{c{k}}}, bw" for k in range(W)] + ["add.cc.u32 {r0}, d0, m0"] + \
            [f"addc.cc.u32 {{r{k}}}, d{k}, m{k}" for k in range(1, W - 1)] + [f"addc.u32 {{r{W-1}}}, d{W-1}, m{W-1}", "}"]
    ins = [("r", f"a[{i}]", f"a{i}") for i in range(W)] + [("r", f"c[{i}]", f"c{i}") for i in range(W)]
    s.append(f"// r = a mod c for a < 2c (one conditional subtraction: c = 2q takes [0, 4q) to [0, 2q), c = q [0, 2q) to [0, q))\n")
    s.append(f"__device__ __forceinline__ void reduce_c{NB}(const uint32_t a[{W}], const uint32_t c[{W}], uint32_t r[{W}]) {{\n"
             + asm_block(lines, outs, ins) + "}\n\n")
    return "".join(s)


def main():
    w6 = ("// ---- 192-bit moduli (6 words, R = 2^192): the same generator at W = 6, used by plans whose\n"
          "// moduli are all < 2^192 (residues still stored in 32-byte slots, top limb zero).\n\n")
    head = ("// arith256_gen.cuh -- GENERATED by tools/gen_arith256.py; do not edit by hand.\n"
            "// 256-bit (8 x 32-bit word) modular arithmetic for sm_100a (SURVEY.md §8(f) f4: wider\n"
            "// multi-word moduli, the paper's stated generalisation, PAPER.md:807-808).  Any odd\n"
            "// q < 2^256; residues canonical (< q) at every interface.  Lazy class (q < 2^254 / 2^190):\n"
            "// values in [0, 4q) between stages, Harvey butterflies (add_nored, sub_add_nored, reduce_c,\n"
            "// mont_mul*_lazy), as the 128-bit LAZY class of arith128.cuh.\n"
            "#pragma once\n#include <cstdint>\n\nnamespace ntt256 {\n\n")
    with open(OUT, "w") as f:
        f.write(head + gen_addsub(8) + gen_mont(8) + gen_lazy(8) + gen_mont(8, True) + w6 +
                gen_addsub(6) + gen_mont(6) + gen_lazy(6) + gen_mont(6, True) + "}  // namespace ntt256\n")
    print("wrote", OUT)


if __name__ == "__main__":
    main()
