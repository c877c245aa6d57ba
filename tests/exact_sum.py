"""Python replay of the device's exact objective accumulator (assign.cu
add_exact): a double is added as a 1088-bit fixed-point integer split in
32-bit limbs; rounding the limb sum once equals math.fsum."""

import numpy as np


def add_exact(s, limbs):
    if s == 0.0:
        return
    bits = np.array([s]).view(np.uint64)[0].item()
    ex = (bits >> 52) & 0x7FF
    m = bits & ((1 << 52) - 1)
    b = 0
    if ex:
        m |= 1 << 52
        b = ex - 1
    idx, sh = b >> 5, b & 31
    sg = -1 if bits >> 63 else 1
    c0 = (m << sh) & 0xFFFFFFFF
    t = (m >> (32 - sh)) if sh else (m >> 32)
    limbs[idx] += sg * c0
    limbs[idx + 1] += sg * (t & 0xFFFFFFFF)
    limbs[idx + 2] += sg * (t >> 32)


def limbs_of(values):
    limbs = [0] * 34
    for s in values:
        add_exact(float(s), limbs)
    return limbs
