# constants for the table exp
from fractions import Fraction
import math, struct
import mpmath
mpmath.mp.prec = 200
ln2_64 = mpmath.log(2)/64
# hi part with 32 significant bits so kd*hi is exact for |kd| < 2^20
def hi_bits(v, bits):
    m, e = math.frexp(float(v))
    m = math.floor(m * 2**bits) / 2**bits
    return math.ldexp(m, e)
hi = hi_bits(ln2_64, 32)
lo = float(ln2_64 - mpmath.mpf(hi))
print("HI", repr(hi), "LO", repr(lo), "INV", repr(float(64/mpmath.log(2))))
tab = [float(mpmath.mpf(2)**(mpmath.mpf(j)/64)) for j in range(64)]
print("TAB", [float.hex(t) for t in tab][:3])
open("tab.h","w").write("static const double TAB[64] = {" + ",".join(float.hex(t) for t in tab) + "};\n" +
  f"#define LN2_64_HI {float.hex(hi)}\n#define LN2_64_LO {float.hex(lo)}\n#define INV_LN2_64 {float.hex(float(64/mpmath.log(2)))}\n")
