"""Multi-rank path on CPU: world_size 2 and 3 over gloo.

Each rank owns a contiguous row shard; the exchange code under test
(paper_2002_09094_b200.dist: statistics all-reduce, row routing to cluster
range owners, mean-slice all-gather) is the production code; the local
compute is the oracle (there is no GPU here).  The sharded run must equal the
single-process oracle run bit for bit: labels, exact objective, means.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from exact_sum import limbs_of


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _dataset(n=900, dim=300, seed=21):
    from paper_2002_09094_b200 import synth

    spec = synth.CONFIGS[0]["corpus"].scaled(n, dim, seed=seed)
    ip, t, v, _ = synth.make_corpus(spec)

    class DS:
        pass

    ds = DS()
    ds.dim, ds.indptr, ds.term_ids, ds.values = dim, ip, t, v
    return ds


def _sims(ds, labels, m):
    """Per-object summands of objective_cosine (clustering.py:105-119)."""
    n = ds.indptr.size - 1
    owners = np.repeat(np.arange(n), np.diff(ds.indptr))
    rows = (labels.astype(np.int64) - 1)[owners]
    mkeys = np.repeat(np.arange(m.k, dtype=np.int64), np.diff(m.indptr)) * (m.dim + 1) + \
        m.term_ids.astype(np.int64)
    ekeys = rows * (m.dim + 1) + ds.term_ids.astype(np.int64)
    pos = np.minimum(np.searchsorted(mkeys, ekeys), mkeys.size - 1)
    hit = mkeys[pos] == ekeys
    contrib = ds.values * np.where(hit, m.values[pos], 0.0)
    return np.bincount(owners, weights=contrib, minlength=n)


def _worker(rank, world, port, k, iters, q):
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2002_09094_b200.dist import (STAT_WORDS, Rows, ShardComm, cluster_range,
                                            pack_stats, shard_rows, unpack_stats)

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = ShardComm(rank, world)
    ds = _dataset()
    lo, hi = shard_rows(ds.indptr, world)[rank]
    a, b = int(ds.indptr[lo]), int(ds.indptr[hi])

    class Shard:
        dim = ds.dim
        indptr = ds.indptr[lo:hi + 1] - a
        term_ids = ds.term_ids[a:b]
        values = ds.values[a:b]

    means = O.init_means(ds, k, 4)
    prev = None
    members = None
    vec = torch.zeros(STAT_WORDS + k, dtype=torch.int64)
    out = []
    for _ in range(iters):
        labels, _, _, post = O.assign(Shard, means)
        sims = _sims(Shard, labels, means)
        changed = 0 if prev is None else int(np.sum(labels != prev))
        sizes = np.bincount(labels - 1, minlength=k)
        # the local statistics in ivfkm_stats' layout (what the kernels write)
        raw = torch.tensor([post, changed, 0, 0, 0, 0] + limbs_of(sims), dtype=torch.int64)
        rows = Rows(torch.from_numpy(Shard.indptr.copy()),
                    torch.from_numpy(Shard.term_ids.astype(np.int32) - 1),
                    torch.from_numpy(Shard.values.copy()),
                    torch.from_numpy(labels.astype(np.int32) - 1))
        prev_t = None if prev is None else torch.from_numpy(prev.astype(np.int32) - 1)
        # DistLloyd.assign: the exchange plan rides on the statistics' one host read
        plan = comm.plan_exchange(rows, prev_t, k, members is None)
        pack_stats(vec, raw, torch.from_numpy(sizes.astype(np.int64)))
        comm.allreduce_sum_(vec)
        h = torch.cat([vec, plan["counts"].reshape(-1), plan["rcounts"].reshape(-1)])
        st = unpack_stats(h[:vec.numel()])
        host = h[vec.numel():].view(2, world, 5).tolist()
        members = comm.exchange_members(members, lo, rows, prev_t, k, plan, host)
        clo, chi = cluster_range(k, world, rank)
        assert bool(torch.all(members.gid[1:] > members.gid[:-1]))  # ascending global order
        assert bool(torch.all((members.labels >= clo) & (members.labels < chi)))

        class Recv:
            dim = ds.dim
            indptr = members.row_ptr.numpy()
            term_ids = members.terms.numpy() + 1
            values = members.vals.numpy()

        p0, p1 = int(means.indptr[clo]), int(means.indptr[chi])
        prev_slice = O.Means(chi - clo, ds.dim, means.indptr[clo:chi + 1] - p0,
                             means.term_ids[p0:p1], means.values[p0:p1],
                             means.retained[clo:chi])
        new = O.update(Recv, members.labels.numpy() - clo + 1, prev_slice)
        ptr, terms, vals, ret = comm.allgather_means(
            torch.from_numpy(new.indptr), torch.from_numpy(new.term_ids - 1),
            torch.from_numpy(new.values), torch.from_numpy(new.retained.astype(np.uint8)))
        # after the first iteration only movers cross: notices + rows of the
        # objects whose owner changed
        if prev is None:
            bound = None
        else:
            from paper_2002_09094_b200.dist import cluster_owner_bounds

            bnd = cluster_owner_bounds(k, world).numpy()
            own_o = np.searchsorted(bnd, prev - 1, side="right")
            own_n = np.searchsorted(bnd, labels - 1, side="right")
            ch = labels != prev
            mv = ch & (own_o != own_n)
            lens = np.diff(Shard.indptr)
            bound = 16 * int(ch.sum()) + int(np.sum(24 + 12 * lens[mv])) + 4 * world
        out.append(dict(labels=labels, post=st["postings"], changed=st["changed"],
                        objective=st["objective"], sizes=vec[STAT_WORDS:].numpy().copy(),
                        sent=comm.last_exchange_bytes, bound=bound))
        means = O.Means(k, ds.dim, ptr.numpy(), terms.numpy().astype(np.int32) + 1,
                        vals.numpy(), ret.numpy().astype(bool))
        prev = labels
    q.put((rank, lo, hi, out, means.indptr, means.term_ids, means.values, means.retained))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,k", [(2, 12), (3, 7), (2, 1), (3, 40)])
def test_sharded_lloyd_equals_single_process(world, k):
    from oracle import oracle as O

    iters = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, k, iters, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ds = _dataset()
    m = O.init_means(ds, k, 4)
    prev = None
    for it in range(iters):
        labels, _, _, post = O.assign(ds, m)
        full = np.concatenate([r[3][it]["labels"] for r in res])
        assert np.array_equal(full, labels), f"labels differ at iteration {it + 1}"
        for r in res:
            assert r[3][it]["post"] == post
            assert r[3][it]["objective"] == O.objective(ds, labels, m)
            assert r[3][it]["changed"] == (0 if prev is None else int(np.sum(labels != prev)))
            assert np.array_equal(r[3][it]["sizes"], O.sizes_of(labels, k))
            if r[3][it]["bound"] is not None:  # only what changed was exchanged
                assert r[3][it]["sent"] <= r[3][it]["bound"], (r[3][it]["sent"],
                                                               r[3][it]["bound"])
        m = O.update(ds, labels, m)
        prev = labels
    for r in res:  # every rank holds the same, bit-identical means
        assert np.array_equal(r[4], m.indptr) and np.array_equal(r[5], m.term_ids)
        assert np.array_equal(r[6], m.values) and np.array_equal(r[7], m.retained)


def test_shard_and_cluster_ranges_cover_everything():
    from paper_2002_09094_b200.dist import cluster_range, shard_rows

    ds = _dataset()
    for world in (1, 2, 3, 8):
        b = shard_rows(ds.indptr, world)
        assert b[0][0] == 0 and b[-1][1] == ds.indptr.size - 1
        assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
        for k in (1, 5, 100):
            r = [cluster_range(k, world, i) for i in range(world)]
            assert r[0][0] == 0 and r[-1][1] == k
            assert all(r[i][1] == r[i + 1][0] for i in range(world - 1))
