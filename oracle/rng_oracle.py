"""CPU restatement of NumPy's PCG64 stream and ziggurat normal sampler -- TEST INFRASTRUCTURE.

Third-party algorithm on the reference path: numpy 2.3.5 ``numpy.random.PCG64`` (PCG XSL-RR
128/64, O'Neill 2014) and ``Generator.standard_normal`` (256-layer ziggurat, Marsaglia & Tsang
2000 with Doornik's tail handling), as called by the reference at leverage.py:124-126,
:196-198 and :217.  This restatement pins the GPU kernels of
paper_2209_04876_b200/csrc/ks_rng.cu: tests check it against NumPy itself and the GPU against
both.  Only tests/ may import it.
"""

from __future__ import annotations

import math

import numpy as np

MASK64 = (1 << 64) - 1
MASK128 = (1 << 128) - 1
PCG_MULT = (0x2360ED051FC65DA4 << 64) | 0x4385DF649FCCF645
ZIG_R = 3.6541528853610087963519472518
ZIG_INV_R = 0.27366123732975827203338247596


def pcg_output(state: int) -> int:
    hi, lo = state >> 64, state & MASK64
    rot = hi >> 58
    x = hi ^ lo
    return ((x >> rot) | (x << ((64 - rot) & 63))) & MASK64


def pcg_advance(state: int, inc: int, delta: int) -> int:
    """Brown's O(log n) LCG jump-ahead."""
    acc_mult, acc_plus, cur_mult, cur_plus = 1, 0, PCG_MULT, inc
    while delta:
        if delta & 1:
            acc_mult = (acc_mult * cur_mult) & MASK128
            acc_plus = (acc_plus * cur_mult + cur_plus) & MASK128
        cur_plus = ((cur_mult + 1) * cur_plus) & MASK128
        cur_mult = (cur_mult * cur_mult) & MASK128
        delta >>= 1
    return (acc_mult * state + acc_plus) & MASK128


def raw_stream(state: int, inc: int, count: int, skip: int = 0):
    s = pcg_advance(state, inc, skip)
    out = np.empty(count, dtype=np.uint64)
    for i in range(count):
        s = (s * PCG_MULT + inc) & MASK128
        out[i] = pcg_output(s)
    return out


def unit(r) -> float:
    return float(int(r) >> 11) * 2.0 ** -53


def standard_normals(raw, tables, count):
    """Ziggurat normals consuming the raw 64-bit stream ``raw``; returns (values, consumed)."""
    ki, wi, fi = tables
    out = np.empty(count)
    q = 0
    for n in range(count):
        while True:
            r = int(raw[q]); q += 1
            idx = r & 0xFF
            r >>= 8
            sign = r & 1
            rabs = (r >> 1) & 0x000FFFFFFFFFFFFF
            x = float(rabs) * float(wi[idx])
            if sign:
                x = -x
            if rabs < int(ki[idx]):
                out[n] = x
                break
            if idx == 0:
                while True:
                    xx = -ZIG_INV_R * math.log1p(-unit(raw[q])); q += 1
                    yy = -math.log1p(-unit(raw[q])); q += 1
                    if yy + yy > xx * xx:
                        v = ZIG_R + xx
                        out[n] = -v if ((rabs >> 8) & 1) else v
                        break
                break
            u = unit(raw[q]); q += 1
            if (float(fi[idx - 1]) - float(fi[idx])) * u + float(fi[idx]) < math.exp(-0.5 * x * x):
                out[n] = x
                break
    return out, q
