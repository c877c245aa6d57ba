"""Golden fixtures for ingestion, made by running the REFERENCE's own io.py
(parse_uci_bow / tfidf_normalize, io.py:72-174) on small inputs:

    python tests/golden/make_golden_io.py

Writes tests/golden/io_cases.json: for every input text either the
reference's ParseError message (with its line number) or its RawCounts and
tf-idf Dataset (values as float.hex, dropped documents, the warning text).
The inputs are the reference tests' hand cases (test_sparse_data.py:56-127)
plus malformed variants and seeded random corpora.
"""

from __future__ import annotations

import io
import json
import sys
import warnings
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from sparse_kmeans import io as rio  # noqa: E402  (the reference package)

OUT = Path(__file__).resolve().parent / "io_cases.json"


def random_bow(n_docs, dim, per_doc, seed, universal=False, blank_lines=False):
    rng = np.random.default_rng(seed)
    lines = []
    for d in range(1, n_docs + 1):
        m = int(rng.integers(1, per_doc + 1))
        p = 1.0 / np.arange(1, dim + 1) ** 1.1
        terms = np.sort(rng.choice(np.arange(1, dim + 1), size=min(m, dim), replace=False,
                                   p=p / p.sum()))
        if universal and 1 not in terms:
            terms = np.sort(np.append(terms, 1))
        for t in terms:
            lines.append(f"{d} {int(t)} {int(rng.geometric(0.4))}")
            if blank_lines and rng.random() < 0.05:
                lines.append("   ")
    order = rng.permutation(len(lines))  # the reference sorts the triples
    body = [lines[i] for i in order]
    n_entries = sum(1 for s in body if s.strip())
    return f"{n_docs}\n{dim}\n{n_entries}\n" + "\n".join(body) + "\n"


CASES = {
    # reference tests (test_sparse_data.py)
    "basic": "2\n3\n3\n1 1 2\n1 3 1\n2 2 5\n",
    "empty_dataset": "0\n0\n0\n",
    "term_out_of_range": "1\n3\n1\n1 4 1\n",
    "duplicate": "1\n3\n2\n1 2 1\n1 2 4\n",
    "nnz_mismatch": "1\n3\n2\n1 2 1\n",
    "empty_input": "",
    "universal_term": "2\n2\n3\n1 1 1\n2 1 1\n2 2 1\n",
    "single_doc_empty": "1\n1\n1\n1 1 3\n",
    "hand_three_docs": "3\n2\n4\n1 1 1\n1 2 1\n2 2 1\n3 2 1\n",
    "unit_norms": "3\n4\n6\n1 1 2\n1 2 1\n2 2 3\n2 3 1\n3 3 2\n3 4 5\n",
    # malformed variants: every error kind, and the first-in-line-order rule
    "header_not_int": "2\nabc\n3\n",
    "header_negative": "2\n-3\n3\n",
    "header_blank": "2\n\n3\n",
    "truncated_header_1": "5\n",
    "truncated_header_2": "5\n7",
    "two_fields": "2\n3\n2\n1 1\n2 2 1\n",
    "four_fields": "2\n3\n2\n1 1 1 1\n2 2 1\n",
    "non_integer": "2\n3\n2\n1 x 1\n2 2 1\n",
    "float_count": "2\n3\n2\n1 1 1.5\n2 2 1\n",
    "doc_zero": "2\n3\n2\n0 1 1\n2 2 1\n",
    "doc_too_big": "2\n3\n2\n3 1 1\n2 2 1\n",
    "term_zero": "2\n3\n2\n1 0 1\n2 2 1\n",
    "count_zero": "2\n3\n2\n1 1 0\n2 2 1\n",
    "count_negative": "2\n3\n2\n1 1 -4\n2 2 1\n",
    "dup_before_error": "2\n3\n4\n1 1 1\n1 1 2\n2 9 1\n2 2 1\n",
    "error_before_dup": "2\n3\n4\n1 1 1\n2 9 1\n1 1 2\n2 2 1\n",
    "dup_later_pair_first": "3\n3\n5\n2 2 1\n1 1 1\n3 3 1\n1 1 5\n2 2 7\n",
    "too_many_entries": "2\n3\n1\n1 1 1\n2 2 1\n",
    "blank_lines_ok": "2\n3\n3\n\n1 1 2\n   \n1 3 1\n2 2 5\n\n",
    "plus_and_underscore": "2\n3\n3\n+1 1 2\n1 3 1_0\n2 0_2 5\n",
    "tabs_crlf": "2\r\n3\r\n3\r\n1\t1\t2\r\n1 3 1\r\n2 2 5\r\n",
    "no_trailing_newline": "2\n3\n3\n1 1 2\n1 3 1\n2 2 5",
    "unordered": "3\n5\n5\n3 5 1\n1 2 2\n2 1 1\n1 1 4\n3 2 2\n",
    # seeded random corpora (shuffled lines; universal term; blank lines)
    "random_small": random_bow(40, 60, 12, 1),
    "random_universal": random_bow(60, 80, 15, 2, universal=True),
    "random_blank": random_bow(50, 70, 10, 3, blank_lines=True),
    "random_medium": random_bow(500, 800, 60, 4),
}


def run(text):
    rec = {"text": text}
    try:
        raw = rio.parse_uci_bow(io.StringIO(text))
    except rio.ParseError as exc:
        rec["parse_error"] = str(exc)
        rec["line"] = exc.line
        return rec
    rec["n_docs"], rec["dim"] = raw.n_docs, raw.dim
    rec["triples"] = [list(t) for t in raw.triples]
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        try:
            ds = rio.tfidf_normalize(raw)
        except ValueError as exc:
            rec["tfidf_error"] = str(exc)
            return rec
    rec["warnings"] = [str(x.message) for x in w]
    rec["indptr"] = [int(x) for x in ds.indptr]
    rec["terms"] = [int(x) for x in ds.term_ids]
    rec["values"] = [float(x).hex() for x in ds.values]
    rec["dropped"] = [int(x) for x in ds.dropped_docs]
    return rec


def main():
    cases = {name: run(text) for name, text in CASES.items()}
    OUT.write_text(json.dumps(cases, indent=0, sort_keys=True) + "\n")
    print(f"wrote {OUT} ({len(cases)} cases)")


if __name__ == "__main__":
    main()
