"""Constants of include/pxg_sincos.h (double sin/cos on the reference's sampler angles).

  python tools/gen/gen_sincos_consts.py   -> prints the C initialisers

pi/2 is split into four doubles (three of 33 significant bits, so q * C_k is exact for the
quadrant counts q < 2^20, and a 53-bit tail); sin(j/64), cos(j/64) for j = 0..52 and the
Taylor coefficients (-1)^k / n! are rounded to double / split into (hi, lo) double pairs.
Computed with mpmath at 300 bits.
"""
import mpmath

mpmath.mp.prec = 300


def split_bits(x, bits):
    """x rounded toward zero to `bits` significant bits (exactly representable)."""
    e = int(mpmath.floor(mpmath.log(abs(x), 2)))
    scale = mpmath.mpf(2) ** (bits - 1 - e)
    return mpmath.floor(x * scale) / scale


def hexd(x):
    return float(x).hex()


def main():
    rest = mpmath.pi / 2
    parts = []
    for bits in (33, 33, 33):
        p = split_bits(rest, bits)
        assert mpmath.mpf(float(p)) == p
        parts.append(p)
        rest -= p
    parts.append(mpmath.mpf(float(rest)))
    print("/* pi/2 = C1 + C2 + C3 + C4 */")
    for i, p in enumerate(parts):
        print(f"#define PXG_SC_C{i + 1} {hexd(p)}")
    print(f"#define PXG_SC_TWO_OVER_PI {hexd(2 / mpmath.pi)}")
    print("/* (-1)^k / n! */")
    for n in (3, 5, 7, 9, 2, 4, 6, 8):
        print(f"#define PXG_SC_F{n} {hexd(mpmath.mpf((-1) ** (n // 2)) / mpmath.factorial(n))}")
    print("/* {sin_hi, sin_lo, cos_hi, cos_lo} of j/64, j = 0..52 */")
    print("#define PXG_SC_TAB_INIT { \\")
    for j in range(53):
        a = mpmath.mpf(j) / 64
        row = []
        for v in (mpmath.sin(a), mpmath.cos(a)):
            hi = mpmath.mpf(float(v))
            row += [hexd(hi), hexd(v - hi)]
        print("  {" + ", ".join(row) + "}, \\")
    print("}")


if __name__ == "__main__":
    main()
