"""TEST INFRASTRUCTURE: the discrete-Gaussian CDT of oracle/bfv_oracle.cpp (kCdt)
and csrc/params.cpp (the device copy), sigma = 3.2, support |x| <= 19 (SEAL's
6-sigma tail cut; the paper's HE library is Pyfhel over SEAL).

    T[k] = floor(2^63 * P(|X| <= k)),  P(X = x) = exp(-x^2 / (2 sigma^2)) / Z,
    Z = sum_{|x| <= 19} exp(-x^2 / (2 sigma^2)),  T[19] = 2^63 (total mass).

The committed table was produced with double-precision arithmetic, so its low
~10 bits are rounding noise of that computation.  This script recomputes the
exact table with 60-digit decimal arithmetic and, with --check, verifies that
every committed entry agrees with it to within 2^-50 (relative to 2^63), which
is the precision the sampler needs (a 2^-50 probability shift is far below any
statistical test of sigma = 3.2).  Run: python oracle/gen_cdt.py [--check]."""
from __future__ import annotations

import re
import sys
from decimal import Decimal, getcontext
from pathlib import Path

SIGMA = Decimal("3.2")
TAIL = 19


def exact_table():
    getcontext().prec = 60
    w = [(-(Decimal(x) ** 2) / (2 * SIGMA * SIGMA)).exp() for x in range(TAIL + 1)]
    z = w[0] + 2 * sum(w[1:])
    out, acc = [], Decimal(0)
    for k in range(TAIL + 1):
        acc += w[k] if k == 0 else 2 * w[k]
        out.append(int((acc / z) * (Decimal(2) ** 63)))
    out[-1] = 1 << 63
    return out


def committed_table():
    src = (Path(__file__).parent / "bfv_oracle.cpp").read_text()
    body = re.search(r"kCdt\[20\]\s*=\s*\{(.*?)\};", src, re.S).group(1)
    return [int(h, 16) for h in re.findall(r"0x([0-9a-fA-F]+)ULL", body)]


def main():
    exact = exact_table()
    if "--check" in sys.argv:
        got = committed_table()
        worst = max(abs(a - b) for a, b in zip(got, exact))
        ok = len(got) == len(exact) and worst < (1 << 13)  # 2^13 / 2^63 = 2^-50
        print(f"max |committed - exact| = {worst} (units of 2^-63): {'ok' if ok else 'MISMATCH'}")
        return 0 if ok else 1
    for i in range(0, len(exact), 4):
        print("    " + ", ".join(f"0x{v:016x}ULL" for v in exact[i:i + 4]) + ",")
    return 0


if __name__ == "__main__":
    sys.exit(main())
