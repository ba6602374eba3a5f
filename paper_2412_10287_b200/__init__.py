"""B200-native single-source two-way regular path queries (arXiv 2412.10287).

Drop-in for the query entry points of the reference package ``rpq``
(/root/reference/pkg/src/rpq/__init__.py): same names, arguments and
exceptions, evaluated by a persistent sm_100a CUDA kernel behind the C ABI in
include/rpq_b200.h.  Graphs and automata are the reference's own
``LabeledGraph`` / ``TwoNfa`` objects (read duck-typed) or the host mirrors
defined here.
"""

from .automaton import Automaton, TransitionTable, reverse, transition_table
from .engine import (
    ALGORITHMS,
    EngineError,
    EngineOptions,
    EvalResult,
    PreparedQuery,
    QueryTimeout,
    eval_sdr,
    eval_ssr,
    eval_ssr_batch,
    eval_ssr_hybrid,
    eval_ssr_masked,
    eval_ssr_no_mask,
    step_update,
)
from .graph import CsrMatrix, DeviceGraph, LabeledGraph, device_graph
from .plan import eval_plan

__all__ = [
    "ALGORITHMS",
    "Automaton",
    "CsrMatrix",
    "DeviceGraph",
    "EngineError",
    "EngineOptions",
    "EvalResult",
    "LabeledGraph",
    "PreparedQuery",
    "QueryTimeout",
    "TransitionTable",
    "device_graph",
    "eval_plan",
    "eval_sdr",
    "eval_ssr",
    "eval_ssr_batch",
    "eval_ssr_hybrid",
    "eval_ssr_masked",
    "eval_ssr_no_mask",
    "reverse",
    "step_update",
    "transition_table",
]
