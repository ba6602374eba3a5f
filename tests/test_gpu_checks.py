"""Memory-safety checks in place of compute-sanitizer (closed on this pool):
the upload rejects malformed CSR structure, and the checked build
(librpq_b200_checked.so, -DRPQ_CHECKED: a bounds check on every
data-dependent device index, csrc/checks.cuh) turns an out-of-range access
into an error naming the site.  The whole GPU suite also runs green on the
checked build (tools/gpu_checked.sh; log under profiles/)."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2412_10287_b200 as P
from paper_2412_10287_b200.graph import CsrMatrix

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_upload_rejects_malformed_csr():
    a_star = P.Automaton.build(1, {(0, False): [(0, 0)]}, [0], [0])
    nv = 100
    bad_col = CsrMatrix(nv, nv, np.array([0, 1] + [1] * (nv - 1), np.int64), np.array([nv + 7], np.int64))
    g = P.LabeledGraph(nv, ["a"], [bad_col], backward=[CsrMatrix(nv, nv, np.zeros(nv + 1, np.int64),
                                                                 np.zeros(0, np.int64))])
    with pytest.raises(ValueError, match="CSR structure invalid"):
        P.eval_ssr(g, a_star, 0, P.EngineOptions(kernel="grid"))
    indptr = np.zeros(nv + 1, np.int64)
    indptr[5:] = 2
    indptr[6] = 1  # decreasing
    indptr[-1] = 2
    bad_ptr = CsrMatrix(nv, nv, indptr, np.array([1, 2], np.int64))
    g2 = P.LabeledGraph(nv, ["a"], [bad_ptr], backward=[bad_ptr])
    with pytest.raises(ValueError, match="CSR structure invalid"):
        P.eval_ssr(g2, a_star, 0, P.EngineOptions(kernel="grid"))


CHILD = r"""
import ctypes, json, math, sys
sys.path.insert(0, sys.argv[1])
import numpy as np, torch
import paper_2412_10287_b200 as P
from paper_2412_10287_b200 import _lib, datagen
lib = _lib.engine()
out = {"checked": lib.rpq_checked_build()}
sg = datagen.generate("cfg1")
g = sg.labeled_graph()
n = P.Automaton.from_json(json.load(open(sys.argv[1] + "/paper_2412_10287_b200/data/config_automata.json"))["cfg1"]["a b*|min"])
r = P.eval_ssr(g, n, 0, P.EngineOptions(timeout=math.inf, kernel="grid"))
out["answer"] = int(r.reach.sum())
# a frontier with a bit past |V| (in the row padding): the step would expand
# vertex |V| + 3, which has no row
pq = P.PreparedQuery(g, n)
w = ctypes.c_int64(); lib.rpq_query_row_words(pq.q, ctypes.byref(w)); W = int(w.value)
m = torch.zeros((n.nstates, W), dtype=torch.int32, device="cuda")
v = sg.nv + 3
m[0, v >> 5] = 1 << (v & 31)
p = torch.zeros_like(m); o = torch.zeros_like(m)
s = torch.cuda.Stream()
rc = lib.rpq_query_step_device(pq.q, m.data_ptr(), p.data_ptr(), o.data_ptr(), s.cuda_stream)
st = _lib.RpqStats()
rc2 = lib.rpq_query_wait(pq.q, ctypes.byref(st)) if rc == 0 else rc
out["step_rc"] = rc2
out["error"] = _lib.last_error()
print(json.dumps(out))
"""


def test_checked_build_reports_out_of_range_access():
    so = os.path.join(ROOT, "paper_2412_10287_b200", "librpq_b200_checked.so")
    if not os.path.exists(so):
        pytest.skip("checked build not present")
    env = dict(os.environ, RPQ_ENGINE="checked")
    res = subprocess.run([sys.executable, "-c", CHILD, ROOT], env=env, capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    out = json.loads(res.stdout.strip().splitlines()[-1])
    assert out["checked"] == 1
    assert out["answer"] == 8869  # cfg1 a b* from 0: the reference's answer (tests/golden/cfg1.json.gz)
    assert out["step_rc"] != 0 and "bounds check failed at ssr_kernel.cuh" in out["error"], out
