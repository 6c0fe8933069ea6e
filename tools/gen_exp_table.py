"""Generate the 2^(k/128) table of the glibc/ARM-optimized-routines exp
algorithm restated in paper_2401_03555_b200/csrc/ndtr.h.

  2^(k/N) ~= H[k] * (1 + T[k]),  H[k] = 2^(k/N) rounded to double,
  T[k] = 2^(k/N) / H[k] - 1 rounded;  tab[2k] = bits(T[k]),
  tab[2k+1] = bits(H[k]) - (k << 52) / N.          (N = 128)

Exact values from Python's decimal module at 80 digits.  Prints C
initialiser lines.
"""
import struct
from decimal import Decimal, getcontext

getcontext().prec = 80
N = 128


def bits(x):
    return struct.unpack("<Q", struct.pack("<d", x))[0]


for k in range(N):
    e = Decimal(2) ** (Decimal(k) / Decimal(N))
    h = float(e)
    t = float((e - Decimal(h)) / Decimal(h))
    hb = (bits(h) - ((k << 52) // N)) & 0xFFFFFFFFFFFFFFFF
    print(f"    0x{bits(t):016x}ull, 0x{hb:016x}ull,")
