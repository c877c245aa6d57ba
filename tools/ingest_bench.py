"""Time ingestion (UCI bag-of-words text -> tf-idf unit vectors) end to end.

    python tools/ingest_bench.py [--docs 300000] [--dim 100000] [--per-doc 230] [--reference]

Builds a seeded docword text in memory (Zipf terms, geometric counts, lines
shuffled), then times parse_uci_bow + tfidf_normalize (native parser on all
host threads, device sort / tf-idf).  ``--reference`` also times the
reference's own io.parse_uci_bow + tfidf_normalize on the same text (only
where /root/reference exists, i.e. not on the GPU box) and checks the two
datasets agree bit for bit.  Prints one JSON line.
"""

import argparse
import io
import json
import sys
import time
import warnings
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def make_text(n_docs, dim, per_doc, seed=11):
    from paper_2002_09094_b200 import synth

    spec = synth.CorpusSpec(n_docs, dim, "poisson", float(per_doc), 0.0, 1, 4 * per_doc, 1.1,
                            seed)
    ip, terms, _, _ = synth.make_corpus(spec)
    n = ip.size - 1
    docs = np.repeat(np.arange(1, n + 1), np.diff(ip))
    rng = np.random.default_rng(seed)
    counts = rng.geometric(0.5, terms.size)
    order = rng.permutation(terms.size)
    body = "\n".join(f"{d} {t} {c}" for d, t, c in
                     zip(docs[order].tolist(), terms[order].tolist(), counts[order].tolist()))
    return f"{n}\n{dim}\n{terms.size}\n{body}\n", terms.size


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--docs", type=int, default=300_000)
    ap.add_argument("--dim", type=int, default=100_000)
    ap.add_argument("--per-doc", type=int, default=230)
    ap.add_argument("--reference", action="store_true")
    a = ap.parse_args()
    import torch

    from paper_2002_09094_b200 import io as pio

    t0 = time.perf_counter()
    text, nnz = make_text(a.docs, a.dim, a.per_doc)
    t_gen = time.perf_counter() - t0
    data = text.encode()
    pio.tfidf_normalize(pio.parse_uci_bow(io.StringIO("2\n3\n3\n1 1 2\n1 3 1\n2 2 5\n")))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hp = pio._parse_host(data)
    t_parse = time.perf_counter() - t0
    t0 = time.perf_counter()
    raw = pio.parse_uci_bow(io.BytesIO(data))
    t_parse_sort = time.perf_counter() - t0
    t0 = time.perf_counter()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        ds = pio.tfidf_normalize(raw)
    torch.cuda.synchronize()
    t_tfidf = time.perf_counter() - t0
    line = {"what": "ingestion: UCI bag-of-words text -> tf-idf Dataset", "docs": a.docs,
            "dim": a.dim, "entries": nnz, "text_bytes": len(data), "gen_s": t_gen,
            "host_parse_s": t_parse, "parse_uci_bow_s": t_parse_sort, "tfidf_normalize_s": t_tfidf,
            "total_s": t_parse_sort + t_tfidf,
            "entries_per_s": nnz / (t_parse_sort + t_tfidf), "n_out": ds.n,
            "host_threads": __import__("os").cpu_count(), "n_read": hp.n_read}
    if a.reference:
        sys.path.insert(0, "/root/reference/pkg/src")
        from sparse_kmeans import io as rio

        t0 = time.perf_counter()
        rraw = rio.parse_uci_bow(io.StringIO(text))
        t_rp = time.perf_counter() - t0
        t0 = time.perf_counter()
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            rds = rio.tfidf_normalize(rraw)
        t_rt = time.perf_counter() - t0
        line.update({"reference_parse_s": t_rp, "reference_tfidf_s": t_rt,
                     "reference_total_s": t_rp + t_rt,
                     "identical": bool(np.array_equal(rds.indptr, ds.indptr)
                                       and np.array_equal(rds.term_ids, ds.term_ids)
                                       and np.array_equal(rds.values.view(np.int64),
                                                          ds.values.view(np.int64)))})
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
