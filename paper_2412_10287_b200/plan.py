"""The plan evaluator (rpq.engine.eval_plan, engine.py:292-390) on the device.

The reference evaluates the regex AST bottom-up with a bound endpoint: a
1 x |V| row vector walked along the AST (`_plan_vector`, engine.py:334-360),
closures as vector fixpoints (`_vec_closure`, :322-331), a destination
binding by walking the reversed AST (query_compiler.py:77-90).  Here the
vector is a device bitmap and every label step `vec x A_l` (bool_matmul,
sparse_bool.py:231-251) is one step of the persistent kernel in step mode
(rpq_query_step_device) on a one-state automaton {0 -l-> 0}, with an empty
visited set, so the step is the plain product (push, or pull when the vector
is dense).  Unions / differences / emptiness are bitmap operations.  The
iteration count and the deadline checks follow the reference call for call:
`state.tick()` per closure round, `clock.check` at every vector step.

The AST is the reference's own (Label / Concat / Alt / Star / Plus / Opt,
query_compiler.py:27-57), read duck-typed by class name and attributes; the
mirror classes below exist for callers without the reference.
"""

import time
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Label:
    name: str
    inverted: bool = False


@dataclass(frozen=True)
class Concat:
    children: tuple


@dataclass(frozen=True)
class Alt:
    children: tuple


@dataclass(frozen=True)
class Star:
    child: object


@dataclass(frozen=True)
class Plus:
    child: object


@dataclass(frozen=True)
class Opt:
    child: object


def ast_from_json(d):
    """Fixture format of tests/golden/make_golden.py (plan cases)."""
    k = d["k"]
    if k == "label":
        return Label(d["name"], bool(d["inv"]))
    if k in ("concat", "alt"):
        kids = tuple(ast_from_json(c) for c in d["c"])
        return Concat(kids) if k == "concat" else Alt(kids)
    return {"star": Star, "plus": Plus, "opt": Opt}[k](ast_from_json(d["c"]))


def _kind(node):
    return type(node).__name__


def reverse_ast(ast):
    """query_compiler.py:77-90: read right-to-left with every symbol inverted."""
    k = _kind(ast)
    if k == "Label":
        return Label(ast.name, not ast.inverted)
    if k == "Concat":
        return Concat(tuple(reverse_ast(c) for c in reversed(ast.children)))
    if k == "Alt":
        return Alt(tuple(reverse_ast(c) for c in ast.children))
    if k == "Star":
        return Star(reverse_ast(ast.child))
    if k == "Plus":
        return Plus(reverse_ast(ast.child))
    if k == "Opt":
        return Opt(reverse_ast(ast.child))
    raise TypeError(f"not a regex node: {ast!r}")


class _Clock:
    """engine.py:80-89: the deadline is checked with the iterations so far."""

    def __init__(self, timeout):
        self.timeout = timeout
        self.t0 = time.monotonic()

    def elapsed(self):
        return time.monotonic() - self.t0

    def check(self, iterations):
        if self.elapsed() > self.timeout:
            from .engine import QueryTimeout

            raise QueryTimeout(self.elapsed(), iterations)


class _DevicePlan:
    """Vector operations of one eval_plan call on the device (one stream)."""

    def __init__(self, g, device, clock):
        import torch

        from .automaton import Automaton
        from .partition import DeviceStep

        self.g = g
        self.nv = int(g.num_vertices)
        self.dev = torch.device("cuda", device)
        self.clock = clock
        self.iterations = 0
        self._steps = {}
        self._Automaton = Automaton
        self._DeviceStep = DeviceStep
        self.stream = torch.cuda.Stream(self.dev)
        probe = self._step_for(None)
        self.words = probe.row_words if probe is not None else ((self.nv + 31) // 32 + 3) // 4 * 4

    def _step_for(self, key):
        """The step kernel of symbol `key` = (label index, inverted); any one
        for key None (to learn the row stride)."""
        if key is None:
            if self.g.num_labels == 0:
                return None
            key = (0, False)
        st = self._steps.get(key)
        if st is None:
            n = self._Automaton.build(1, {key: [(0, 0)]}, [0], [0])
            st = self._DeviceStep(self.g, n, self.dev)
            self._steps[key] = st
        return st

    def zeros(self):
        import torch

        return torch.zeros((1, self.words), dtype=torch.int32, device=self.dev)

    def nnz(self, v):
        return bool(v.any())

    def tick(self):
        self.iterations += 1
        self.clock.check(self.iterations)

    def label(self, node, vec):
        """vec x A_l (or A_l^T): bool_matmul(vec, _plan_adjacency(node))."""
        ids = getattr(self.g, "label_ids", None)
        if ids is None:
            ids = {name: i for i, name in enumerate(self.g.labels)}
        if node.name not in ids:  # engine.py:284-287: unknown label -> zero matrix
            return self.zeros()
        st = self._step_for((ids[node.name], bool(node.inverted)))
        out, p = self.zeros(), self.zeros()  # P empty: the plain product
        st(vec, p, out, self.stream.cuda_stream)
        return out

    def vector(self, node, vec):
        """_plan_vector (engine.py:334-360)."""
        self.clock.check(self.iterations)
        if not self.nnz(vec):
            return vec
        k = _kind(node)
        if k == "Label":
            return self.label(node, vec)
        if k == "Concat":
            for child in node.children:
                vec = self.vector(child, vec)
            return vec
        if k == "Alt":
            acc = self.vector(node.children[0], vec)
            for child in node.children[1:]:
                acc = acc | self.vector(child, vec)
            return acc
        if k == "Star":
            return self.closure(vec, node.child)
        if k == "Plus":
            return self.closure(self.vector(node.child, vec), node.child)
        if k == "Opt":
            return vec | self.vector(node.child, vec)
        raise TypeError(f"not a regex node: {node!r}")

    def closure(self, vec, child):
        """_vec_closure (engine.py:322-331): vec x child* as a fixpoint."""
        acc = vec
        frontier = vec
        while self.nnz(frontier):
            self.tick()
            frontier = self.vector(child, frontier) & ~acc
            acc = acc | frontier
        return acc

    def close(self):
        for st in self._steps.values():
            st.close()


def eval_plan(g, ast, endpoint, opts=None):
    """rpq.engine.eval_plan (engine.py:363-390) on the device: the answer set
    reached from (endpoint = ("source", v)) or reaching (("destination", v))
    the bound vertex, iterations = closure rounds."""
    import torch

    from .engine import EngineOptions, EvalResult, _check_vertex

    opts = opts or EngineOptions()
    opts.validate()
    mode, vertex = endpoint
    if mode == "destination":
        ast = reverse_ast(ast)
    elif mode != "source":
        raise ValueError(f"endpoint mode must be source or destination, got {mode!r}")
    _check_vertex(g, vertex)
    clock = _Clock(opts.timeout)
    plan = _DevicePlan(g, opts.device, clock)
    try:
        with torch.cuda.stream(plan.stream):
            start = plan.zeros()
            start[0, vertex >> 5] = np.array([1 << (vertex & 31)], dtype=np.uint32).view(np.int32)[0].item()
            result = plan.vector(ast, start)
            words = result[0].cpu().numpy().view(np.uint32)
    finally:
        plan.close()
    nw = (plan.nv + 31) // 32
    return EvalResult(None, plan.iterations, clock.elapsed(), "plan", bits=np.ascontiguousarray(words[:nw]),
                      nv=plan.nv)
