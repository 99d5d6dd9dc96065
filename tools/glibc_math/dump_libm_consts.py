"""Dev tool: print the FP64 constants glibc 2.39's x86-64 libm uses in erf and in the
FMA variant of exp, read from the installed libm.so.6 at the addresses its disassembly
loads them from (objdump -d, erf@@GLIBC_2.2.5 at 0x2df70, __exp_fma at 0x79b60).

The constants are the published fdlibm s_erf.c coefficients and the table/poly data of
the 2018 table-driven exp (EXP_TABLE_BITS = 7); this script only confirms their exact
bits so csrc/glibc_math.cuh can restate them. Not used at build or run time.
"""
import math
import struct
import sys

LIBM = "/lib/x86_64-linux-gnu/libm.so.6"

ERF_ADDRS = {
    "efx16": 0x99A80, "sixteen": 0x99A38, "sixteenth": 0x98FA0, "dbl_min": 0x98EE0,
    "efx": 0x99A88, "one": 0x98E18,
    # |x| < 0.84375
    "s0_a": 0x99A90, "s0_b": 0x99A98, "s0_c": 0x99AA0, "s0_d": 0x99AA8, "s0_e": 0x99AB0,
    "s0_f": 0x99AB8, "s0_g": 0x99AC0, "s0_h": 0x99AC8, "s0_i": 0x99AD0, "s0_j": 0x99AD8,
    # 0.84375 <= |x| < 1.25
    "s1_a": 0x99AE0, "s1_b": 0x99AE8, "s1_c": 0x99AF0, "s1_d": 0x99AF8, "s1_e": 0x99B00,
    "s1_f": 0x99B08, "s1_g": 0x99B10, "s1_h": 0x99B18, "s1_i": 0x99B20, "s1_j": 0x99B28,
    "s1_k": 0x99B30, "s1_l": 0x99B38, "s1_m": 0x99B40, "erx": 0x99B48, "nerx": 0x99B50,
    "tiny": 0x99B58,
    # 1.25 <= |x| < 1/0.35
    "s2_a": 0x99B60, "s2_b": 0x99B68, "s2_c": 0x99B70, "s2_d": 0x99B78, "s2_e": 0x99B80,
    "s2_f": 0x99B88, "s2_g": 0x99B90, "s2_h": 0x99B98, "s2_i": 0x99BA0, "s2_j": 0x99BA8,
    "s2_k": 0x99BB0, "s2_l": 0x99BB8, "s2_m": 0x99BC0, "s2_n": 0x99BC8, "s2_o": 0x99BD0,
    "s2_p": 0x99BD8,
    # 1/0.35 <= |x| < 6
    "s3_a": 0x99BE0, "s3_b": 0x99BE8, "s3_c": 0x99BF0, "s3_d": 0x99BF8, "s3_e": 0x99C00,
    "s3_f": 0x99C08, "s3_g": 0x99C10, "s3_h": 0x99C18, "s3_i": 0x99C20, "s3_j": 0x99C28,
    "s3_k": 0x99C30, "s3_l": 0x99C38, "s3_m": 0x99C40, "s3_n": 0x99C48, "c0p5625": 0x99C50,
}
EXP_ADDRS = {
    "invln2N": 0xB4980, "shift": 0xB4988, "negln2hiN": 0xB4990, "negln2loN": 0xB4998,
    "C2": 0xB49A0, "C3": 0xB49A8, "C4": 0xB49B0, "C5": 0xB49B8, "two1009": 0x98FF8,
}
EXP_TAB = 0xB4A30  # __exp_data.tab, 2*128 uint64


def load():
    with open(LIBM, "rb") as f:
        return f.read()


def u64(blob, vaddr):  # the read-only segments of this libm map vaddr == file offset
    return struct.unpack_from("<Q", blob, vaddr)[0]


def main():
    blob = load()
    out = sys.stdout
    for name, addrs in (("erf", ERF_ADDRS), ("exp", EXP_ADDRS)):
        for k, a in addrs.items():
            b = u64(blob, a)
            d = struct.unpack("<d", struct.pack("<Q", b))[0]
            out.write(f"{name} {k:10s} 0x{b:016x}  {d!r}\n")
    tab = [u64(blob, EXP_TAB + 8 * i) for i in range(256)]
    # Check the table against its construction: tab[2i+1] = bits(2^(i/128)) - (i << 45),
    # tab[2i] = bits of the rounding tail (2^(i/128) - s) / s.
    import mpmath
    mpmath.mp.prec = 200
    bad = 0
    for i in range(128):
        v = mpmath.mpf(2) ** (mpmath.mpf(i) / 128)
        s = float(v)
        sb = struct.unpack("<Q", struct.pack("<d", s))[0]
        tail = float((v - mpmath.mpf(s)) / mpmath.mpf(s))
        tb = struct.unpack("<Q", struct.pack("<d", tail))[0]
        if ((sb - (i << 45)) & (2**64 - 1)) != tab[2 * i + 1] or tb != tab[2 * i]:
            bad += 1
    out.write(f"exp table entries not matching the construction: {bad}\n")
    for i in range(0, 256, 4):
        out.write("    " + ", ".join(f"0x{t:016x}ULL" for t in tab[i:i + 4]) + ",\n")


if __name__ == "__main__":
    main()
