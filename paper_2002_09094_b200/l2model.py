"""The reference's last-level-cache model (reference cache.py:1-215),
re-parameterised for the B200 L2 and the BIVF layout.

The reference models an idealised fully associative LRU cache: scanning an
object touches each term p's mean postings with probability no_p / N, a
term's postings cost ceil(nc_p * gamma) cache blocks, z consecutive scans
touch sum_p (1 - (1 - no_p/N)^z) * blocks_p blocks, z* is the largest window
that fits the cache, and a scan misses on term p when p went unseen for z*
objects:  misses = N * sum_p (no_p/N) (1 - no_p/N)^z* * blocks_p
(cache.py:89-215).  Same closed forms here; what changes is what a "block" is:

* the cache is the 126 MB L2 with 32-byte sectors (the DRAM transfer unit);
* a term's block count is the sectors of its BIVF screen data — the fp16
  value run of its spans (dense spans 512 B, sparse spans their padded
  postings) plus the mask and offset words of the spans outside its dense
  prefix — read straight from the built headers (``term_sectors``), instead
  of ceil(nc_p * 12 B / 64 B).

``predict_dram_bytes`` turns the miss count into DRAM bytes per screen launch
(tools/l2_model_report.py sets it beside the ncu-measured dram__bytes_read).
The object rows themselves stream once per launch and are not modelled (as in
the reference, which models the postings only).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = ["CacheParams", "FreqProfile", "expected_blocks_ivf", "expected_blocks_ivf_window",
           "find_z_star", "llcm_ivf", "term_sectors", "predict_dram_bytes"]

K_DENSE = 0x80000000
K_SPAN = 8


@dataclass(frozen=True)
class CacheParams:
    """B200 L2 geometry (cache.py:26-46 with the GPU's numbers): 126 MB in
    32-byte sectors, ``usable`` of it assumed available to posting data (the
    rest holds the streaming object rows and headers in flight)."""

    cache_bytes: int = 126 * 2**20
    block_bytes: int = 32
    usable: float = 0.75

    @property
    def nb_llc(self) -> float:
        return self.usable * self.cache_bytes / self.block_bytes


@dataclass(frozen=True)
class FreqProfile:
    """no_p (objects holding term p) and blocks_p (sectors of p's posting data)
    over N objects (cache.py:49-95, with blocks in place of nc)."""

    no: np.ndarray
    blocks: np.ndarray
    n: int

    def __post_init__(self):
        no = np.ascontiguousarray(self.no, dtype=np.float64)
        bl = np.ascontiguousarray(self.blocks, dtype=np.float64)
        if no.shape != bl.shape or no.ndim != 1:
            raise ValueError("no and blocks must be parallel 1-D arrays")
        if self.n < 1:
            raise ValueError("n must be >= 1")
        if no.size and (no.min() < 0 or no.max() > self.n):
            raise ValueError("no_p must lie in 0..n")
        object.__setattr__(self, "no", no)
        object.__setattr__(self, "blocks", bl)


def expected_blocks_ivf(p: FreqProfile) -> float:
    """Blocks one object's scan pulls: sum_p (no_p/N) blocks_p (cache.py:98-102)."""
    return float(np.dot(p.no / p.n, p.blocks))


def expected_blocks_ivf_window(p: FreqProfile, z) -> float:
    """Distinct blocks of z consecutive scans (cache.py:115-133)."""
    if z == 0:
        return 0.0
    if z == 1:
        return expected_blocks_ivf(p)
    if z < 0:
        raise ValueError("z must be nonnegative")
    if math.isinf(z):
        return float(p.blocks[p.no > 0].sum())
    return float(np.dot(1.0 - (1.0 - p.no / p.n) ** z, p.blocks))


def find_z_star(p: FreqProfile, c: CacheParams):
    """Largest z whose window fits the usable L2 (cache.py:136-163): inf when
    everything reachable fits, 0 when a single scan overflows."""
    if float(p.blocks[p.no > 0].sum()) <= c.nb_llc:
        return math.inf
    if expected_blocks_ivf(p) > c.nb_llc:
        return 0
    hi = 1
    while expected_blocks_ivf_window(p, hi) <= c.nb_llc:
        hi *= 2
    lo = hi // 2
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if expected_blocks_ivf_window(p, mid) <= c.nb_llc:
            lo = mid
        else:
            hi = mid
    return lo


def llcm_ivf(p: FreqProfile, c: CacheParams, z_star=None) -> float:
    """Expected misses (blocks) of one pass over the N objects
    (cache.py:188-215): N * sum_p (no_p/N)(1 - no_p/N)^z* blocks_p, with a
    term's first touch counted once when everything fits."""
    if z_star is None:
        z_star = find_z_star(p, c)
    frac = p.no / p.n
    if math.isinf(z_star):
        return float(p.blocks[p.no > 0].sum())  # compulsory misses only
    return p.n * float(np.dot(frac * (1.0 - frac) ** z_star, p.blocks))


def term_sectors(headers: np.ndarray, k: int, dim: int, nblk: int, value_bytes: int = 2,
                 block_bytes: int = 32) -> np.ndarray:
    """Sectors of each term's screen data from the BIVF headers (bivf.cuh):
    the term's value run [offs[t*nblk], offs[(t+1)*nblk]) in value_bytes each,
    plus 64 B of masks + offsets per span outside the dense prefix dpre[t]."""
    h = np.asarray(headers).view(np.uint32)
    nh = dim * nblk
    offs = h[nh: 2 * nh + 1].astype(np.int64) & ~K_DENSE
    starts = offs[0: nh: nblk]
    ends = np.append(starts[1:], offs[nh])
    nc = h[2 * nh + 1: 2 * nh + 1 + dim]
    dpre = h[2 * nh + 1 + dim + 2 * k: 2 * nh + 1 + dim + 2 * k + dim].astype(np.int64)
    spans = nblk // K_SPAN
    vals = (ends - starts) * value_bytes
    hdr = np.where(nc > 0, (spans - np.minimum(dpre, spans)) * 64, 0)
    return np.ceil(vals / block_bytes) + np.ceil(hdr / block_bytes)


def predict_dram_bytes(no: np.ndarray, blocks: np.ndarray, n: int,
                       params: CacheParams = CacheParams()) -> dict:
    """Modelled DRAM bytes of one screen launch, with z* and the window."""
    p = FreqProfile(no, blocks, n)
    z = find_z_star(p, params)
    misses = llcm_ivf(p, params, z)
    return {"z_star": z, "blocks_per_scan": expected_blocks_ivf(p),
            "reachable_bytes": float(p.blocks[p.no > 0].sum()) * params.block_bytes,
            "dram_bytes": misses * params.block_bytes}
