"""CPU tests that pin the oracle (test infrastructure) to the reference:
hand-computed known answers from the reference's own tests, and golden
vectors the reference itself produced (tests/golden/make_golden.py)."""

import hashlib

import numpy as np
import pytest

from conftest import R, golden_dataset, load_golden
from oracle import oracle as O

SMALL = ["small_k8", "small_k32", "small_k128", "signed_k16", "dups_k40",
         "small_k32_ivfd", "signed_k16_ivfd", "signed_k4_ivfd"]


def _tiny():
    class DS:
        dim = 4
        indptr = np.array([0, 2, 4, 6], np.int64)
        term_ids = np.array([1, 2, 2, 3, 3, 4], np.int32)
        values = np.full(6, R)

    return DS


def _tiny_means():
    s = 6 ** -0.5
    return O.Means(2, 4, np.array([0, 3, 5], np.int64), np.array([1, 2, 3, 3, 4], np.int32),
                   np.array([s, 2 * s, s, R, R]), np.zeros(2, bool))


def test_oracle_assign_tiny_known_answer():
    """test_variants.py:34-39: labels [1,1,2], mults 8 = 1 + 2 + 4 + 1."""
    labels, top1, top2, post = O.assign(_tiny(), _tiny_means())
    assert labels.tolist() == [1, 1, 2]
    assert post == 8 == O.volume_ivf(_tiny(), _tiny_means())
    # x2 against mu1: 0.7071*0.81650 + 0.7071*0.40825 = 0.86603 beats 0.5
    assert top1[1] == pytest.approx(0.86603, abs=1e-5)


def test_oracle_no_overlap_goes_to_cluster_one():
    """test_variants.py:42-50."""
    labels, _, _, post = O.assign_ivf(np.array([0, 1]), np.array([4], np.int32), np.array([1.0]),
                                      np.array([0, 1, 2, 2, 2]), np.array([1, 2], np.int32),
                                      np.array([1.0, 1.0]), 2)
    assert labels.tolist() == [1] and post == 0


def test_oracle_update_tiny():
    """test_variants.py:169-179 / test_clustering_core.py:109-115."""
    ds = _tiny()
    prev = O.Means(2, 4, np.array([0, 2, 4]), np.array([1, 2, 3, 4], np.int32), np.full(4, R),
                   np.zeros(2, bool))
    up = O.update(ds, np.array([1, 1, 2], np.int32), prev)
    s = 6 ** -0.5
    np.testing.assert_allclose(up.values, [s, 2 * s, s, R, R], atol=1e-12)
    ip, own, val = O.inverted(up)
    assert own[ip[2]:ip[3]].tolist() == [1, 2]
    assert val[ip[2]] == pytest.approx(0.40825, abs=1e-5)


def test_oracle_update_empty_cluster_retains():
    """test_variants.py:212-217."""
    up = O.update(_tiny(), np.array([1, 1, 1], np.int32), _tiny_means())
    assert up.retained.tolist() == [False, True]
    assert up.values[up.indptr[1]:].tolist() == _tiny_means().values[3:].tolist()


def test_oracle_objective_hand_value():
    """test_clustering_core.py:76-79: 2.5."""
    m = O.Means(2, 4, np.array([0, 2, 4]), np.array([1, 2, 3, 4], np.int32), np.full(4, R),
                np.zeros(2, bool))
    assert O.objective(_tiny(), np.array([1, 1, 2]), m) == pytest.approx(2.5, abs=1e-12)


def test_fnv1a64_known_answers():
    """test_clustering_core.py:201-204."""
    assert O.clib().oracle_fnv1a64(None, 0) == 0xCBF29CE484222325
    from paper_2002_09094_b200.types import fnv1a64

    assert fnv1a64(b"") == 0xCBF29CE484222325
    assert fnv1a64(b"a") == 0xAF63DC4C8601EC8C


@pytest.mark.parametrize("name", SMALL)
def test_oracle_run_matches_reference_golden(name):
    g = load_golden(name)
    ds = golden_dataset(g)
    variant = str(g["variant"]) if "variant" in g else "IVF"
    res = O.run_ivf(ds, int(g["k"]), int(g["seed"]), max_iter=int(g["max_iter"]),
                    variant=variant)
    assert len(res.iters) == int(g["iterations"])
    assert res.converged == bool(g["converged"])
    for i, it in enumerate(res.iters):
        assert np.array_equal(it.labels, g["labels"][i])
        assert it.objective == float(g["objectives"][i])
        assert it.digest == int(g["digests"][i])
        assert it.postings == int(g["mults"][i]) == int(g["volume_ivf"][i])
        assert it.mean_terms_total == int(g["mean_terms_total"][i])
    assert np.array_equal(res.final_means.indptr, g["final_indptr"])
    assert np.array_equal(res.final_means.term_ids, g["final_terms"])
    assert np.array_equal(res.final_means.values, g["final_values"])
    assert np.array_equal(res.final_means.retained, g["final_retained"])


def test_oracle_run_matches_reference_config0():
    from paper_2002_09094_b200 import synth

    g = load_golden("config0")
    c0 = synth.CONFIGS[0]
    ip, t, v, _ = synth.make_corpus(c0["corpus"])
    h = hashlib.sha256()
    for a in (ip, t, v):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == str(g["inputs_sha"])

    class DS:
        dim = c0["corpus"].dim
        indptr, term_ids, values = ip, t, v

    res = O.run_ivf(DS, c0["k"], c0["seed"], max_iter=c0["iters"], threads=O.host_threads())
    assert len(res.iters) == int(g["iterations"])
    for i, it in enumerate(res.iters):
        assert it.digest == int(g["digests"][i])
        assert it.objective == float(g["objectives"][i])
        assert it.postings == int(g["mults"][i])
    fm = res.final_means
    h = hashlib.sha256()
    for a in (fm.indptr, fm.term_ids, fm.values, fm.retained):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == str(g["final_sha"])


def test_oracle_c_matches_reference_compiled_kernel():
    """The C restatement vs the reference's own Cython kernel (oracle/_ref)."""
    ref = O.ref_kernels()
    if ref is None:
        pytest.skip("oracle/_ref not built (reference not present)")
    from paper_2002_09094_b200 import synth

    spec = synth.CONFIGS[1]["corpus"].scaled(600, 3000, seed=77)
    ip, t, v, _ = synth.make_corpus(spec)

    class DS:
        dim = 3000
        indptr, term_ids, values = ip, t, v

    m = O.init_means(DS, 40, 5)
    mi = O.inverted(m)
    lab, _, _, post = O.assign_ivf(ip, t, v, *mi, 40, threads=3)
    lab_ref = np.empty(ip.size - 1, np.int32)
    ctr = np.zeros(5, np.int64)
    ref.assign_ivf(ip, t, v, mi[0], mi[1], mi[2], np.zeros(40), lab_ref, ctr)
    assert np.array_equal(lab, lab_ref)
    assert post == ctr[0] == ctr[1] == ctr[2]


def test_sample_without_replacement_matches_literal():
    """The product's O(k) Fisher-Yates equals the reference's literal one."""
    from paper_2002_09094_b200.clustering import sample_without_replacement

    for n, k, seed in [(10, 10, 0), (1000, 17, 3), (300000, 1000, 1), (5, 1, 9)]:
        assert np.array_equal(sample_without_replacement(n, k, seed),
                              O.sample_without_replacement(n, k, seed))


@pytest.mark.parametrize("n,dim,k,seed,signed", [(1500, 400, 64, 0, False),
                                                 (3000, 5000, 300, 1, True),
                                                 (2000, 129, 1500, 2, False),
                                                 (600, 4097, 40, 3, True)])
def test_oracle_update_fast_equals_update(n, dim, k, seed, signed):
    """update_fast (vectorised, used at configs 1-4) is bit-identical to the
    literal per-cluster restatement of variants.py:254-307, empty clusters
    and cancelling signed sums included."""
    from oracle import oracle as O
    from paper_2002_09094_b200 import Dataset, synth

    spec = synth.CONFIGS[0]["corpus"].scaled(n, dim, seed=100 + seed)
    ip, t, v, _ = synth.make_corpus(spec)
    if signed:
        v = v * np.where(np.random.default_rng(seed).random(v.size) < 0.4, -1.0, 1.0)
    ds = Dataset(dim, ip, t, v, normalized=True)
    m = O.init_means(ds, min(k, ds.n), seed)
    lab = np.random.default_rng(seed).integers(1, m.k + 1, size=ds.n).astype(np.int32)
    lab[lab == 2] = 1  # an empty cluster
    a = O.update(ds, lab, m)
    b = O.update_fast(ds, lab, m, chunk_bytes=1 << 20)  # several dense chunks
    for f in ("indptr", "term_ids", "values", "retained"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
