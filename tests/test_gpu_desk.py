"""The reference's desk-scale benchmark (test_acceptance.py criterion 7,
:238-335) and its determinism check (criterion 8, :338-369), replayed on the
device: the same generated graph (1e5 vertices, ~1e6 edges, the test's label
skew) and the same 1,000 entries (10 query families x {ssr, sdr} x 50
endpoints), every answer and every algorithm's iteration count compared with
the reference's own (tests/golden/desk_bench.json.gz, make_golden.py desk)."""

import hashlib
import math

import numpy as np
import pytest

from fixtures import answer_digest, automaton, desk_bench, desk_host_graph

import paper_2412_10287_b200 as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def desk():
    rec, csr = desk_bench()
    g = desk_host_graph(rec, csr)
    autos = {pat: automaton(nj) for pat, nj in rec["automata"].items()}
    return rec, g, autos


@pytest.mark.parametrize("algorithm", ["masked", "no_mask", "hybrid"])
def test_desk_bench_answers(desk, algorithm):
    rec, g, autos = desk
    opts = P.EngineOptions(algorithm=algorithm, timeout=60.0)
    for e in rec["entries"]:
        n = autos[e["pattern"]]
        res = P.eval_ssr(g, n, e["vertex"], opts) if e["mode"] == "ssr" else P.eval_sdr(g, n, e["vertex"], opts)
        assert int(res.reach.sum()) == e["count"] and answer_digest(res.reach) == e["sha256"], e["id"]
        assert res.iterations == e["iterations"][algorithm], (e["id"], res.iterations)
        assert res.algorithm == algorithm


def test_desk_bench_determinism(desk):
    """Criterion 8: the hybrid results' bytes are identical run to run, on
    the grid kernel as on the single-CTA one, and equal the reference's."""
    rec, g, autos = desk

    def result_bytes(kernel, direction):
        opts = P.EngineOptions(algorithm="hybrid", timeout=math.inf, kernel=kernel, direction=direction)
        chunks = []
        for e in rec["entries"]:
            n = autos[e["pattern"]]
            f = P.eval_ssr if e["mode"] == "ssr" else P.eval_sdr
            res = f(g, n, e["vertex"], opts)
            chunks.append(f"{e['id']}:" + ",".join(str(v) for v in np.flatnonzero(res.reach).tolist()))
        return hashlib.sha256("\n".join(chunks).encode()).hexdigest()

    for kernel, direction in (("auto", "auto"), ("grid", "auto"), ("grid", "pull"), ("grid", "push")):
        assert result_bytes(kernel, direction) == rec["criterion8_sha256"], (kernel, direction)


def test_desk_bench_batch(desk):
    """Each (family, mode) combination's 50 endpoints through eval_ssr_batch."""
    rec, g, autos = desk
    groups = {}
    for e in rec["entries"]:
        groups.setdefault((e["pattern"], e["mode"]), []).append(e)
    for (pattern, mode), entries in groups.items():
        n = autos[pattern] if mode == "ssr" else P.reverse(autos[pattern])
        rows = P.eval_ssr_batch(g, n, [e["vertex"] for e in entries], P.EngineOptions(timeout=math.inf))
        for e, row in zip(entries, rows):
            assert answer_digest(row) == e["sha256"], e["id"]
