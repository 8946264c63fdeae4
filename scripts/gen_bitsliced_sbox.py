"""Generate a bitsliced AES S-box circuit (tower field GF(((2^2)^2)^2)) as
straight-line CUDA over 8 bit-planes, verified exhaustively before writing.

    python scripts/gen_bitsliced_sbox.py            # writes paper_1403_7295_b200/csrc/sbox_bitsliced.inc
    python scripts/gen_bitsliced_sbox.py --check    # verify the committed file is what this script emits

Construction: the input byte is mapped (8x8 GF(2) matrix T) into the tower
representation a = ah*Y + al over GF(16) = GF(4)[Z]/(Z^2+Z+mu), GF(4) =
GF(2)[w]/(w^2+w+1); the inverse is
    d = lambda*ah^2 + ah*al + al^2,  a^-1 = (ah*d^-1) Y + ((ah+al)*d^-1),
with GF(16) inversion done the same way one level down (GF(4) inverse =
square).  The output map A*T^-1 (AES affine matrix times the inverse
isomorphism) and the constant 0x63 finish SubBytes.  Every gate is a 2-input
XOR / AND (or an XOR with all-ones for the constant); nvcc fuses chains of
them into LOP3.

Verification: the program is executed on 256-bit integers whose bit x is the
value of a wire for input byte x, and compared with the S-box table.
"""
from __future__ import annotations

import argparse
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "paper_1403_7295_b200", "csrc", "sbox_bitsliced.inc")


# ------------------------------------------------------------ GF(2^8) (AES)
def gmul(a, b):
    p = 0
    while b:
        if b & 1:
            p ^= a
        a = ((a << 1) ^ (0x1B if a & 0x80 else 0)) & 0xFF
        b >>= 1
    return p


def aes_sbox():
    inv = [0] * 256
    for x in range(1, 256):
        for y in range(1, 256):
            if gmul(x, y) == 1:
                inv[x] = y
                break
    s = []
    for x in range(256):
        b = inv[x]
        r = b
        for k in range(1, 5):
            r ^= ((b << k) | (b >> (8 - k))) & 0xFF
        s.append(r ^ 0x63)
    return s


# ------------------------------------------------------------ tower field (numeric)
# GF(4): 2-bit (g1 g0) = g1*w + g0, w^2 = w + 1
def m4(a, b):
    a1, a0, b1, b0 = a >> 1, a & 1, b >> 1, b & 1
    hh = a1 & b1
    return ((hh ^ (a1 & b0) ^ (a0 & b1)) << 1) | (hh ^ (a0 & b0))


# GF(16) = GF(4)[Z]/(Z^2 + Z + MU): 4-bit (h<<2)|l
def m16(a, b, MU):
    ah, al, bh, bl = a >> 2, a & 3, b >> 2, b & 3
    hh = m4(ah, bh)
    return ((hh ^ m4(ah, bl) ^ m4(al, bh)) << 2) | (m4(hh, MU) ^ m4(al, bl))


# GF(256) = GF(16)[Y]/(Y^2 + Y + LAM): 8-bit (h<<4)|l
def m256(a, b, MU, LAM):
    ah, al, bh, bl = a >> 4, a & 15, b >> 4, b & 15
    hh = m16(ah, bh, MU)
    return ((hh ^ m16(ah, bl, MU) ^ m16(al, bh, MU)) << 4) | (m16(hh, LAM, MU) ^ m16(al, bl, MU))


def find_tower():
    for MU in range(1, 4):  # Z^2+Z+MU irreducible over GF(4)
        if any(m4(z, z) ^ z ^ MU == 0 for z in range(4)):
            continue
        for LAM in range(1, 16):
            if any(m16(y, y, MU) ^ y ^ LAM == 0 for y in range(16)):
                continue
            # a root beta of the AES polynomial x^8+x^4+x^3+x+1 in the tower field
            for beta in range(2, 256):
                pw = [1]
                for _ in range(8):
                    pw.append(m256(pw[-1], beta, MU, LAM))
                if pw[8] ^ pw[4] ^ pw[3] ^ pw[1] ^ pw[0] == 0:
                    return MU, LAM, pw[:8]
    raise RuntimeError("no tower representation found")


def mat_from_columns(cols):
    """8x8 GF(2) matrix M (list of row bitmasks) with M * e_i = cols[i]."""
    return [sum(((cols[i] >> r) & 1) << i for i in range(8)) for r in range(8)]


def mat_apply(M, x):
    return sum((bin(M[r] & x).count("1") & 1) << r for r in range(8))


def mat_inv(M):
    n = 8
    A = [(M[r], 1 << r) for r in range(n)]
    for c in range(n):
        piv = next(r for r in range(c, n) if (A[r][0] >> c) & 1)
        A[c], A[piv] = A[piv], A[c]
        for r in range(n):
            if r != c and (A[r][0] >> c) & 1:
                A[r] = (A[r][0] ^ A[c][0], A[r][1] ^ A[c][1])
    return [A[r][1] for r in range(n)]


# ------------------------------------------------------------ circuit builder
class Circuit:
    def __init__(self):
        self.lines = []
        self.n = 0
        self.vals = {}
        self.gates = {"xor": 0, "and": 0, "not": 0}

    def new(self, expr, val, kind):
        name = f"t{self.n}"
        self.n += 1
        self.lines.append(f"const uint32_t {name} = {expr};")
        self.vals[name] = val
        self.gates[kind] += 1
        return name

    def xor(self, a, b):
        return self.new(f"{a} ^ {b}", self.vals[a] ^ self.vals[b], "xor")

    def and_(self, a, b):
        return self.new(f"{a} & {b}", self.vals[a] & self.vals[b], "and")

    def not_(self, a):
        return self.new(f"~{a}", self.vals[a] ^ ((1 << 256) - 1), "not")

    def xor_many(self, xs):
        acc = xs[0]
        for x in xs[1:]:
            acc = self.xor(acc, x)
        return acc

    def linear(self, M, ins):
        """outputs r = XOR of ins[i] with M[r] bit i (list indexed by bit)."""
        outs = []
        for r in range(len(M)):
            terms = [ins[i] for i in range(len(ins)) if (M[r] >> i) & 1]
            outs.append(self.xor_many(terms) if len(terms) > 1 else terms[0])
        return outs

    # GF(4) on (g1, g0)
    def gf4_mul(self, a, b):
        a1, a0 = a
        b1, b0 = b
        hh = self.and_(a1, b1)
        ll = self.and_(a0, b0)
        s = self.and_(self.xor(a1, a0), self.xor(b1, b0))  # Karatsuba: (a1+a0)(b1+b0)
        # g1 = a1b1 + a1b0 + a0b1 = s + ll ; g0 = a1b1 + a0b0 = hh + ll
        return (self.xor(s, ll), self.xor(hh, ll))

    def gf4_scale(self, a, c):
        """multiply by constant c in GF(4) (linear)."""
        a1, a0 = a
        if c == 1:
            return a
        if c == 2:  # w*(a1 w + a0) = a1 w^2 + a0 w = a1(w+1) + a0 w = (a1+a0) w + a1
            return (self.xor(a1, a0), a1)
        if c == 3:  # (w+1)*a = w a + a
            t = self.gf4_scale(a, 2)
            return (self.xor(t[0], a1), self.xor(t[1], a0))
        raise ValueError(c)

    def gf4_sq(self, a):
        a1, a0 = a  # (a1 w + a0)^2 = a1 w^2 + a0 = a1 w + (a1 + a0)
        return (a1, self.xor(a1, a0))

    # GF(16) on (h=(g1,g0), l=(g1,g0))
    def gf16_mul(self, a, b, MU):
        ah, al = a
        bh, bl = b
        hh = self.gf4_mul(ah, bh)
        ll = self.gf4_mul(al, bl)
        s = self.gf4_mul((self.xor(ah[0], al[0]), self.xor(ah[1], al[1])),
                         (self.xor(bh[0], bl[0]), self.xor(bh[1], bl[1])))
        h = (self.xor(s[0], ll[0]), self.xor(s[1], ll[1]))          # ah bl + al bh + ah bh = s + ll
        m = self.gf4_scale(hh, MU)
        l = (self.xor(m[0], ll[0]), self.xor(m[1], ll[1]))          # MU ah bh + al bl
        return (h, l)

    def gf16_inv(self, a, MU):
        ah, al = a
        # e = MU ah^2 + ah al + al^2 ; e^-1 = e^2 ; res = (ah e^-1, (ah+al) e^-1)
        t1 = self.gf4_scale(self.gf4_sq(ah), MU)
        t2 = self.gf4_mul(ah, al)
        t3 = self.gf4_sq(al)
        e = (self.xor_many([t1[0], t2[0], t3[0]]), self.xor_many([t1[1], t2[1], t3[1]]))
        ei = self.gf4_sq(e)
        s = (self.xor(ah[0], al[0]), self.xor(ah[1], al[1]))
        return (self.gf4_mul(ah, ei), self.gf4_mul(s, ei))


def gf16_lin_sq_scale(c: Circuit, a, MU, LAM):
    """LAM * a^2 in GF(16) as a linear map of the 4 input bits."""
    bits = [a[1][1], a[1][0], a[0][1], a[0][0]]  # bit0 = l.g0, bit1 = l.g1, bit2 = h.g0, bit3 = h.g1

    def f(x):
        return m16(m16(x, x, MU), LAM, MU)

    M = mat_from_columns([f(1 << i) for i in range(4)] + [0] * 4)[:4]
    M = [row & 0xF for row in M]
    o = c.linear(M, bits)
    return ((o[3], o[2]), (o[1], o[0]))


def build():
    sbox = aes_sbox()
    MU, LAM, betas = find_tower()
    T = mat_from_columns(betas)              # AES bit basis -> tower bits
    Tinv = mat_inv(T)
    A = [0] * 8                              # AES affine matrix rows
    for r in range(8):
        for k in range(5):
            A[r] |= 1 << ((r - k) % 8)
    # out = A * Tinv * y  (as one 8x8 matrix)
    AT = [0] * 8
    for r in range(8):
        for i in range(8):
            col = mat_apply(Tinv, 1 << i)
            if bin(A[r] & col).count("1") & 1:
                AT[r] |= 1 << i

    c = Circuit()
    x = [f"x{i}" for i in range(8)]
    for i in range(8):
        c.vals[x[i]] = sum(((v >> i) & 1) << v for v in range(256))
    y = c.linear(T, x)                       # tower bits: y[7..4] = ah, y[3..0] = al
    ah = ((y[7], y[6]), (y[5], y[4]))
    al = ((y[3], y[2]), (y[1], y[0]))
    # d = LAM ah^2 + ah al + al^2
    t1 = gf16_lin_sq_scale(c, ah, MU, LAM)
    t2 = c.gf16_mul(ah, al, MU)
    t3 = gf16_lin_sq_scale(c, al, MU, 1)
    d = tuple(tuple(c.xor_many([t1[i][j], t2[i][j], t3[i][j]]) for j in range(2)) for i in range(2))
    di = c.gf16_inv(d, MU)
    s = tuple(tuple(c.xor(ah[i][j], al[i][j]) for j in range(2)) for i in range(2))
    ih = c.gf16_mul(ah, di, MU)
    il = c.gf16_mul(s, di, MU)
    inv_bits = [il[1][1], il[1][0], il[0][1], il[0][0], ih[1][1], ih[1][0], ih[0][1], ih[0][0]]
    out = c.linear(AT, inv_bits)
    outs = []
    for r in range(8):
        outs.append(c.not_(out[r]) if (0x63 >> r) & 1 else out[r])
    # verify on all 256 inputs
    for v in range(256):
        got = sum(((c.vals[outs[r]] >> v) & 1) << r for r in range(8))
        assert got == sbox[v], (v, got, sbox[v])
    return c, outs, MU, LAM


def emit(c, outs, MU, LAM):
    body = "\n".join("  " + ln for ln in c.lines)
    assign = "\n".join(f"  x{r} = {outs[r]};" for r in range(8))
    g = c.gates
    return f"""// GENERATED by scripts/gen_bitsliced_sbox.py -- do not edit.
// Bitsliced AES S-box over 8 bit-planes (x0 = bit 0 of every byte), tower
// field GF(((2^2)^2)^2) with MU={MU}, LAMBDA={LAM}; {g['xor']} XOR + {g['and']} AND + {g['not']} NOT
// 2-input gates before nvcc's LOP3 fusion.  Verified on all 256 inputs.
__device__ __forceinline__ void sbox_bitsliced(uint32_t& x0, uint32_t& x1, uint32_t& x2, uint32_t& x3, uint32_t& x4,
                                               uint32_t& x5, uint32_t& x6, uint32_t& x7) {{
{body}
{assign}
}}
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--check", action="store_true")
    args = ap.parse_args()
    c, outs, MU, LAM = build()
    text = emit(c, outs, MU, LAM)
    if args.check:
        ok = os.path.exists(OUT) and open(OUT).read() == text
        print("up to date" if ok else "STALE")
        sys.exit(0 if ok else 1)
    with open(OUT, "w") as f:
        f.write(text)
    print("wrote", OUT, c.gates)


if __name__ == "__main__":
    main()
