"""Ingestion (reference io.py:72-174) against fixtures made by the reference
itself (tests/golden/make_golden_io.py -> io_cases.json).

CPU: the native parser's header/line checks and line numbering (every error
the host decides).  GPU: parse_uci_bow + tfidf_normalize end to end —
messages, sorted triples, tf-idf values bit for bit, dropped documents and
the warning.
"""

from __future__ import annotations

import io
import json
import warnings
from pathlib import Path

import numpy as np
import pytest

GOLD = json.loads((Path(__file__).parent / "golden" / "io_cases.json").read_text())
CPU_DECIDED = [name for name, c in GOLD.items()
               if "parse_error" in c and "duplicate" not in c["parse_error"]]


@pytest.mark.parametrize("name", CPU_DECIDED)
def test_host_parser_errors_match_reference(name):
    from paper_2002_09094_b200 import io as pio

    case = GOLD[name]
    hp = pio._parse_host(case["text"].encode("utf-8"))
    with pytest.raises(pio.ParseError) as ei:
        pio._raise_header(hp)
        pio._raise_body(hp)
    assert str(ei.value) == case["parse_error"]
    assert ei.value.line == case["line"]


@pytest.mark.parametrize("name", [n for n, c in GOLD.items() if "triples" in c])
def test_host_parser_reads_every_valid_triple(name):
    from paper_2002_09094_b200 import io as pio

    case = GOLD[name]
    hp = pio._parse_host(case["text"].encode("utf-8"))
    pio._raise_header(hp)
    pio._raise_body(hp)
    got = sorted(zip(hp.docs[:hp.n_read].tolist(), hp.terms[:hp.n_read].tolist(),
                     hp.counts[:hp.n_read].tolist()))
    assert [list(t) for t in got] == case["triples"]
    assert (int(hp.header[0]), int(hp.header[1])) == (case["n_docs"], case["dim"])


def test_host_parser_threads_agree_on_a_large_buffer():
    """> 1 MiB bodies are split over threads at line boundaries: same triples,
    same line numbers and the same first error as one thread."""
    from paper_2002_09094_b200 import io as pio

    rng = np.random.default_rng(7)
    n = 120_000
    docs = rng.integers(1, 5000, n)
    terms = rng.integers(1, 3000, n)
    body = "\n".join(f"{d} {t} {c}" for d, t, c in zip(docs, terms, rng.integers(1, 9, n)))
    text = f"5000\n3000\n{n}\n{body}\n".encode()
    one = pio._parse_host(text, threads=1)
    many = pio._parse_host(text, threads=8)
    assert one.n_read == many.n_read == n and one.err_line == many.err_line == -1
    for a in ("docs", "terms", "counts", "lines"):
        assert np.array_equal(getattr(one, a)[:n], getattr(many, a)[:n])
    lines = text.split(b"\n")
    lines[90_000] = b"7 7"
    bad = b"\n".join(lines)
    e1, e8 = pio._parse_host(bad, threads=1), pio._parse_host(bad, threads=8)
    assert e1.err_line == e8.err_line == 90_001 and e1.err_code == e8.err_code == 3


# ---------------------------------------------------------------- GPU


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(GOLD))
def test_ingestion_matches_reference(name):
    from paper_2002_09094_b200 import io as pio

    case = GOLD[name]
    if "parse_error" in case:
        with pytest.raises(pio.ParseError) as ei:
            pio.parse_uci_bow(io.StringIO(case["text"]))
        assert str(ei.value) == case["parse_error"] and ei.value.line == case["line"]
        return
    raw = pio.parse_uci_bow(io.StringIO(case["text"]))
    assert (raw.n_docs, raw.dim) == (case["n_docs"], case["dim"])
    assert [list(t) for t in raw.triples] == case["triples"]
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        ds = pio.tfidf_normalize(raw)
    assert [str(x.message) for x in w] == case["warnings"]
    assert ds.indptr.tolist() == case["indptr"]
    assert ds.term_ids.tolist() == case["terms"]
    assert [float(v).hex() for v in ds.values] == case["values"]  # bit for bit
    assert list(ds.dropped_docs) == case["dropped"]


@pytest.mark.gpu
def test_ingested_corpus_runs_through_the_lloyd_path(tmp_path):
    """load_uci_bow from a file feeds run() directly (the reference CLI's
    ingest -> run)."""
    from paper_2002_09094_b200 import io as pio
    from paper_2002_09094_b200.clustering import run

    p = tmp_path / "docword.txt"
    p.write_text(GOLD["random_medium"]["text"])
    ds = pio.load_uci_bow(p)
    assert ds.n == len(GOLD["random_medium"]["indptr"]) - 1
    res = run("IVF", ds, 8, seed=3, max_iter=5)
    assert res.iterations >= 1
