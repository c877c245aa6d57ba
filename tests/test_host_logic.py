"""CPU tests: the C-ABI library loads and exports every declared symbol, the
host-side numerics the kernels implement (pairwise-norm replay, exact
objective accumulator, error window) are right, the mirrored types validate
like the reference, and the generator follows its spec."""

import math
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


# ---------------------------------------------------------------- C ABI

def _declared_symbols():
    text = (ROOT / "include" / "ivfkm.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ivfkm_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2002_09094_b200 import _lib

    lib = _lib.load()
    declared = _declared_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    # the ctypes table binds exactly the header's entry points
    assert sorted(_lib.SIGNATURES) == declared


def test_abi_constants_and_struct_layout():
    import ctypes

    from paper_2002_09094_b200 import _lib

    lib = _lib.load()
    text = (ROOT / "include" / "ivfkm.h").read_text()
    assert f"#define IVFKM_OBJ_LIMBS {_lib.IVFKM_OBJ_LIMBS}" in text
    assert f"#define IVFKM_MAXC {_lib.IVFKM_MAXC}" in text
    assert ctypes.sizeof(_lib.Stats) == 6 * 8 + 8 * _lib.IVFKM_OBJ_LIMBS
    assert lib.ivfkm_version() >= 1
    assert lib.ivfkm_error_string(-4) == b"workspace too small"
    assert lib.ivfkm_bivf_nblk(100) == 8 and lib.ivfkm_bivf_nblk(1000) == 32
    assert lib.ivfkm_bivf_nblk(60000) == 1880
    assert lib.ivfkm_assign_workspace_size(1000, 10) > 1000 * 4 * 36
    assert lib.ivfkm_update_workspace_size(10, 100, 5, 50) > 0
    assert lib.ivfkm_update_state_size(10, 100, 5, 50) > 0
    assert lib.ivfkm_update_state_size(1 << 30, 100, 1 << 20, 1 << 20) == 0  # 70-bit key


def test_host_entry_point_reports_missing_gpu_or_range():
    """ivfkm_assign_ivf_host validates ids like the reference (data.py:261-262)."""
    import ctypes

    from paper_2002_09094_b200 import _lib

    lib = _lib.load()
    ip = np.array([0, 1], np.int64)
    t = np.array([9], np.int32)  # term 9 > dim 4
    v = np.array([1.0])
    mp = np.array([0, 0, 0, 0, 0], np.int64)
    lab = np.zeros(1, np.int32)
    ctr = np.zeros(5, np.int64)
    P = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
    rc = lib.ivfkm_assign_ivf_host(1, P(ip), P(t), P(v), 4, P(mp), None, None, 2, P(lab), P(ctr))
    assert rc in (-5, -6)  # no GPU here, or the range error when one is present


# ---------------------------------------------------------------- numerics replays

def _leaves(D):
    out = []
    stack = [(0, D)]
    while stack:
        lo, n = stack.pop()
        if n <= 128:
            out.append((lo, n))
            continue
        n2 = n // 2
        n2 -= n2 % 8
        stack.append((lo + n2, n - n2))
        stack.append((lo, n2))
    return out


def _leaf_value(lo, n, pos, w2):
    sel = (pos >= lo) & (pos < lo + n)
    p, x = pos[sel], w2[sel]
    if n < 8:
        res = 0.0
        for val in x:
            res += val
        return res
    lim = lo + n - n % 8
    r = [0.0] * 8
    res_tail = []
    for pi, val in zip(p, x):
        if pi < lim:
            r[(pi - lo) & 7] += val
        else:
            res_tail.append(val)
    res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
    for val in res_tail:
        res += val
    return res


def _combine(D, vals):
    it = iter(vals)

    def pw(n):
        if n <= 128:
            return next(it)
        n2 = n // 2
        n2 -= n2 % 8
        a = pw(n2)
        b = pw(n - n2)
        return a + b

    return pw(D)


@pytest.mark.parametrize("D", [1, 5, 7, 8, 100, 128, 129, 1000, 10_000, 100_000, 141_000])
def test_pairwise_norm_replay_matches_numpy(D):
    """The norm kernel's leaf/combine replay equals np.sum(w*w) bit for bit
    (variants.py:298 computes nrm = np.sqrt(np.sum(w * w)))."""
    rng = np.random.default_rng(D)
    for density in (0.001, 0.05, 0.6):
        w = np.zeros(D)
        m = rng.random(D) < density
        w[m] = rng.random(m.sum()) / 7.0
        pos = np.flatnonzero(w)
        w2 = w[pos] * w[pos]
        vals = [_leaf_value(lo, n, pos, w2) for lo, n in _leaves(D)]
        assert _combine(D, vals) == float(np.sum(w * w))


from exact_sum import add_exact as _add_exact  # noqa: E402


def test_exact_objective_accumulator_equals_fsum():
    """The fixed-point superaccumulator, rounded once on the host, is math.fsum
    (clustering.py:119)."""
    from paper_2002_09094_b200.engine import objective_from_limbs

    rng = np.random.default_rng(1)
    cases = [rng.random(5000), rng.random(2000) ** 9 - 0.3, np.array([1e-300, 1.0, -1.0]),
             np.array([5e-324, 2.0 ** -1022, 0.75]), np.array([3.9, -3.9, 1e-17])]
    for x in cases:
        limbs = [0] * 34
        for s in x:
            _add_exact(float(s), limbs)
        assert objective_from_limbs(limbs) == math.fsum(x.tolist())


def test_error_window_is_rigorous():
    """|rho32 - rho64| stays inside the kernel's eps_i on adversarial-ish rows."""
    rng = np.random.default_rng(2)
    for n in (1, 10, 230, 2000):
        for _ in range(20):
            v = rng.random(n)
            v /= np.linalg.norm(v)
            u = rng.random(n) * (rng.random(n) < 0.7)
            u /= max(np.linalg.norm(u), 1e-300)
            acc32 = np.float32(0)
            for a, b in zip(v.astype(np.float32), u.astype(np.float32)):
                acc32 = np.float32(np.fma(a, b, acc32)) if hasattr(np, "fma") else \
                    np.float32(np.float64(a) * np.float64(b) + np.float64(acc32))
            acc64 = 0.0
            for a, b in zip(v, u):
                acc64 = acc64 + a * b
            eps = ((n + 3) * 2.0 ** -24 + n * 2.0 ** -50) * (1 + 1e-9) * (1 + 1e-6) + \
                (n + 1) * 2.0 ** -125
            assert abs(float(acc32) - acc64) <= eps


def test_fp16_error_window_is_rigorous():
    """The fp16 screen (mean values rounded to fp16, object values to fp32,
    fp32 FMAs in any order) stays inside its eps_i (csrc/assign.cu,
    screen_epilogue) — including values below fp16's normal
    range, signed data, and the worst accumulation order (largest first)."""
    rng = np.random.default_rng(3)
    for n in (1, 10, 230, 2000):
        for trial in range(24):
            v = 10.0 ** rng.uniform(-7 if trial % 3 == 0 else -2, 0, n)
            u = 10.0 ** rng.uniform(-7 if trial % 2 == 0 else -2, 0, n) * (rng.random(n) < 0.7)
            if trial % 4 == 1:  # signed
                v *= np.where(rng.random(n) < 0.5, -1.0, 1.0)
                u *= np.where(rng.random(n) < 0.5, -1.0, 1.0)
            v /= np.linalg.norm(v)
            u /= max(np.linalg.norm(u), 1e-300)
            order = np.argsort(-np.abs(v * u)) if trial % 2 else rng.permutation(n)
            v32, u16 = v.astype(np.float32), u.astype(np.float16).astype(np.float32)
            # the screen sums dense-span products in registers and sparse-span
            # products in a slot scratch, then folds the scratch in: two
            # partial fp32 sums and one more rounding (trial % 3 == 2)
            parts = [order] if trial % 3 != 2 else [order[::2], order[1::2]]
            accs = []
            for part in parts:
                acc32 = np.float32(0)
                for h in part:
                    acc32 = np.float32(np.float64(v32[h]) * np.float64(u16[h]) + np.float64(acc32))
                accs.append(acc32)
            acc32 = accs[0] if len(accs) == 1 else np.float32(np.float64(accs[0]) + np.float64(accs[1]))
            acc64 = 0.0
            for a, b in zip(v, u):
                acc64 = acc64 + a * b
            xn, mu = float(np.linalg.norm(v)), 1.0
            eps = (2.0 ** -11 + (n + 5) * 2.0 ** -24) * xn * mu * (1 + 2.0 ** -9) + \
                n * xn * 2.0 ** -25 * (1 + 2.0 ** -9) + (n + 1) * 2.0 ** -125
            assert abs(float(acc32) - acc64) <= eps, (n, trial, abs(float(acc32) - acc64), eps)


# ---------------------------------------------------------------- types

def test_types_validate_like_reference():
    from paper_2002_09094_b200 import Assignment, Dataset, MeanSet

    with pytest.raises(ValueError, match="malformed indptr"):
        Dataset(4, np.array([1, 2]), np.array([1], np.int32), np.array([1.0]))
    with pytest.raises(ValueError, match="1..dim"):
        Dataset(4, np.array([0, 1]), np.array([5], np.int32), np.array([1.0]))
    with pytest.raises(ValueError, match="strictly increasing"):
        Dataset(4, np.array([0, 2]), np.array([2, 2], np.int32), np.array([0.6, 0.8]))
    with pytest.raises(ValueError, match="non-unit"):
        Dataset(4, np.array([0, 1]), np.array([1], np.int32), np.array([0.5]), normalized=True)
    with pytest.raises(ValueError, match="unit L2"):
        MeanSet.from_csr(np.array([0, 1]), np.array([1], np.int32), np.array([0.5]), 4)
    with pytest.raises(ValueError, match="1..k"):
        Assignment(np.array([0, 1]), np.array([1, 1]))
    a = Assignment.from_labels(np.array([1, 1, 2]), 3)
    assert a.sizes.tolist() == [2, 1, 0] and a.n == 3 and a.k == 3
    assert not a.labels.flags.writeable


def test_init_means_matches_oracle(tiny):
    from oracle import oracle as O
    from paper_2002_09094_b200.clustering import init_means

    m = init_means(tiny, 2, seed=5, representation="sparse_inverted")
    o = O.init_means(tiny, 2, 5)
    assert np.array_equal(m.indptr, o.indptr) and np.array_equal(m.term_ids, o.term_ids)
    assert np.array_equal(m.values, o.values)
    with pytest.raises(ValueError):
        init_means(tiny, 4, seed=1)


# ---------------------------------------------------------------- generator

def test_synth_deterministic_and_well_formed():
    from paper_2002_09094_b200 import Dataset, synth

    spec = synth.CONFIGS[1]["corpus"].scaled(3000, 20000, seed=3)
    a = synth.make_corpus(spec)
    b = synth.make_corpus(spec)
    for x, y in zip(a[:3], b[:3]):
        assert np.array_equal(x, y)
    ip, t, v, dropped = a
    ds = Dataset(spec.dim, ip, t, v, normalized=True)  # validates 1-based, increasing, unit
    rows = np.diff(ip)
    assert rows.min() >= 1 and rows.max() <= 2000
    assert 150 < rows.mean() < 320  # lognormal mean 230, clipped
    assert np.all(v > 0)
    df = ds.doc_freq
    # Zipf: the most frequent kept term is a top-ranked one; a term in every
    # row has idf 0 and is dropped (df == N never survives, io.py:153-154)
    assert df.max() < ds.n and int(np.argmax(df)) < 5


def test_synth_config_shapes():
    from paper_2002_09094_b200 import synth

    c = synth.CONFIGS
    assert (c[0]["corpus"].n, c[0]["corpus"].dim, c[0]["k"]) == (20000, 10000, 100)
    assert (c[1]["corpus"].n, c[1]["corpus"].dim, c[1]["k"]) == (300000, 100000, 1000)
    assert c[2]["corpus"] is c[1]["corpus"] and c[2]["k"] == 10000
    assert (c[3]["corpus"].n, c[3]["corpus"].dim, c[3]["k"]) == (8200000, 141000, 10000)
    assert c[4]["corpus"] is c[3]["corpus"] and c[4]["k"] == 60000


def test_row_gap_encoding_round_trips():
    """encode_row_gaps (the end-to-end upload's 16-bit term gaps): decoding
    with a plain cumulative sum per row (exceptions absolute) restores every
    id, including rows that start beyond 0xFFFF and gaps of exactly 0xFFFF."""
    from paper_2002_09094_b200.engine import encode_row_gaps

    rng = np.random.default_rng(3)
    dim = 300_000
    rows = [np.sort(rng.choice(dim, m, replace=False)) for m in rng.integers(0, 40, 200)]
    rows += [np.array([0xFFFE, 0xFFFE + 0xFFFF, 0xFFFE + 2 * 0xFFFF + 1]), np.array([70000]),
             np.array([], dtype=np.int64), np.array([0, 1, 2])]
    ip = np.zeros(len(rows) + 1, np.int64)
    np.cumsum([r.size for r in rows], out=ip[1:])
    terms0 = np.concatenate(rows).astype(np.int32)
    gaps, exc_idx, exc_term = encode_row_gaps(ip, terms0)
    assert gaps.dtype == np.uint16 and exc_idx.size == exc_term.size > 0
    out = np.empty_like(terms0)
    exc = dict(zip(exc_idx.tolist(), exc_term.tolist()))
    for i in range(len(rows)):
        cur = -1
        for h in range(ip[i], ip[i + 1]):
            cur = exc[h] if gaps[h] == 0xFFFF else cur + int(gaps[h])
            out[h] = cur
    assert np.array_equal(out, terms0)


def test_l2_model_closed_forms():
    """l2model (reference cache.py restated for the B200 L2): the window at
    z=1 is one scan, the window is monotone in z, z* is the last fitting
    window, everything fitting leaves the compulsory misses only, and a
    smaller cache misses more."""
    import math

    from paper_2002_09094_b200 import l2model as L

    rng = np.random.default_rng(5)
    no = rng.integers(0, 500, 300)
    blocks = rng.integers(1, 40, 300).astype(float)
    p = L.FreqProfile(no, blocks, 500)
    assert L.expected_blocks_ivf_window(p, 1) == L.expected_blocks_ivf(p)
    w = [L.expected_blocks_ivf_window(p, z) for z in (1, 2, 4, 8, 16)]
    assert all(a <= b for a, b in zip(w, w[1:]))
    c = L.CacheParams(cache_bytes=int(w[2] * 32 / 0.75) + 64, block_bytes=32, usable=0.75)
    z = L.find_z_star(p, c)
    assert L.expected_blocks_ivf_window(p, z) <= c.nb_llc < L.expected_blocks_ivf_window(p, z + 1)
    big = L.CacheParams(cache_bytes=10**9)
    assert math.isinf(L.find_z_star(p, big))
    assert L.llcm_ivf(p, big) == blocks[no > 0].sum()
    assert L.llcm_ivf(p, c) > L.llcm_ivf(p, big)


@pytest.mark.parametrize("k,passes,rowcap", [(1000, 1, 512), (10000, 10, 512), (10000, 5, 128),
                                             (60000, 30, 128)])
def test_screen_plan_keeps_nine_ctas_under_the_196k_carveout(k, passes, rowcap):
    """The screen's loads allocate L1 lines while in flight, and the L1 is what
    the shared-memory carve-out leaves of 256 KB: nine CTAs (the register
    limit at 56 registers x 128 threads) must fit the 196 KB carve-out, or
    the driver moves to 228 KB and the screen loses a quarter of its speed
    (DESIGN.md section 4a).  Plans of BASELINE configs 1-4 (host-side query)."""
    from paper_2002_09094_b200 import _lib

    lib = _lib.load()
    out = np.zeros(8, np.int32)
    lib.ivfkm_set_tuning(rowcap, -1, 0)
    lib.ivfkm_set_screen_option(1, passes)
    try:
        _lib.check(lib.ivfkm_screen_plan(k, rowcap, 16, out.ctypes.data), "plan")
    finally:
        lib.ivfkm_set_screen_option(1, 0)
        lib.ivfkm_set_tuning(1024, -1, 0)
    warps, dyn, maxreg = int(out[3]), int(out[6]), int(out[7])
    assert warps <= 4 and maxreg == 56
    static_and_reserved = 1200 + 1024  # ScreenShared, counters; 1 KB per CTA for the driver
    assert 9 * (dyn + static_and_reserved) <= 196 * 1024, (dyn, warps)
