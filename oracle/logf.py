"""Natural logarithm in fp32, transcribed operation by operation from the
FreeBSD msun `e_logf.c` algorithm (argument reduction x = 2^k (1+f) with
sqrt(2)/2 < 1+f < sqrt(2); s = f/(2+f); log(1+f) = f - s(f - R(s^2)) with the
degree-4 Lg polynomial), every operation IEEE round-to-nearest-even on fp32
and no fused multiply-add.  TEST INFRASTRUCTURE ONLY (oracle/__init__.py).

SURVEY §8(c) O-S fixes this algorithm for the Gumbel noise g = -LOG(-LOG(u))
so that CPU and GPU samplers agree bit for bit; numpy float32 element-wise
operations are single IEEE operations, so this vectorised transcription
rounds exactly like the scalar C code evaluated left to right.

The algorithm follows FreeBSD msun e_logf.c, which carries this notice:
  Conversion to float by Ian Lance Taylor, Cygnus Support, ian@cygnus.com.
  ====================================================
  Copyright (C) 1993 by Sun Microsystems, Inc. All rights reserved.

  Developed at SunPro, a Sun Microsystems, Inc. business.
  Permission to use, copy, modify, and distribute this
  software is freely granted, provided that this notice
  is preserved.
  ====================================================
"""
from __future__ import annotations

import numpy as np

F = np.float32
LN2_HI = F(6.9313812256e-01)   # 0x3f317180
LN2_LO = F(9.0580006145e-06)   # 0x3717f7d1
TWO25 = F(3.355443200e+07)     # 0x4c000000
LG1 = F(0xAAAAAA * 2.0 ** -24)  # 0.66666662693
LG2 = F(0xCCCE13 * 2.0 ** -25)  # 0.40000972152
LG3 = F(0x91E9EE * 2.0 ** -25)  # 0.28498786688
LG4 = F(0xF89E26 * 2.0 ** -26)  # 0.24279078841
THIRD = F(0.33333333333333333)  # (float)0.333... in the source
HALF = F(0.5)
ONE = F(1.0)
TWO = F(2.0)


def logf(x) -> np.ndarray:
    x = np.atleast_1d(np.asarray(x, dtype=np.float32)).copy()
    ix = x.view(np.int32).copy()
    out = np.full(x.shape, np.nan, dtype=np.float32)
    done = np.zeros(x.shape, dtype=bool)
    with np.errstate(all="ignore"):
        k = np.zeros(x.shape, dtype=np.int32)
        tiny = ix < 0x00800000
        zero = (ix & 0x7FFFFFFF) == 0
        out[zero] = -np.inf
        done |= zero
        neg = tiny & (ix < 0) & ~zero
        out[neg] = np.nan
        done |= neg
        sub = tiny & ~zero & ~neg
        k = np.where(sub, k - 25, k)
        x = np.where(sub, x * TWO25, x).astype(np.float32)
        ix = x.view(np.int32).copy()
        big = (ix >= 0x7F800000) & ~done
        out[big] = (x + x)[big]
        done |= big

        k = k + ((ix >> 23) - 127)
        ix = ix & 0x007FFFFF
        i = (ix + (0x95F64 << 3)) & 0x800000
        x = (ix | (i ^ 0x3F800000)).astype(np.int32).view(np.float32)
        k = k + (i >> 23)
        f = x - ONE
        dk = k.astype(np.float32)

        small = ((0x007FFFFF & (0x8000 + ix)) < 0xC000) & ~done
        # -2^-9 <= f < 2^-9
        fz = small & (f == F(0.0))
        r = np.where(k == 0, F(0.0), dk * LN2_HI + dk * LN2_LO)
        out[fz] = r[fz]
        R = f * f * (HALF - THIRD * f)
        r = np.where(k == 0, f - R, dk * LN2_HI - ((R - dk * LN2_LO) - f))
        sel = small & ~fz
        out[sel] = r[sel]
        done |= small

        s = f / (TWO + f)
        z = s * s
        i2 = ix - (0x6147A << 3)
        w = z * z
        j = (0x6B851 << 3) - ix
        t1 = w * (LG2 + w * LG4)
        t2 = z * (LG1 + w * LG3)
        i2 = i2 | j
        R = t2 + t1
        hfsq = HALF * f * f
        r_pos = np.where(k == 0, f - (hfsq - s * (hfsq + R)),
                         dk * LN2_HI - ((hfsq - (s * (hfsq + R) + dk * LN2_LO)) - f))
        r_neg = np.where(k == 0, f - s * (f - R), dk * LN2_HI - ((s * (f - R) - dk * LN2_LO) - f))
        r = np.where(i2 > 0, r_pos, r_neg)
        rest = ~done
        out[rest] = r[rest]
    return out.astype(np.float32)
