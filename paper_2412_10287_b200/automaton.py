"""Query automata: the reference's ``TwoNfa`` read duck-typed, a host mirror
type, and the transition table the device kernel consumes.

The engine reads a compiled automaton exactly the way the reference engine
does (rpq/engine.py:92-109): it iterates ``sorted(n.alphabet)`` -- not
``n.transitions`` -- skips symbols whose label index is not a graph label
(engine.py:100-101), looks each symbol's matrix up in ``n.transitions`` (a
KeyError there is the reference's behaviour too), and seeds from
``n.start_set``; answers are projected through ``n.final_set``.
"""

import hashlib
from dataclasses import dataclass, field

import numpy as np

from .graph import CsrMatrix


def _matrix_pairs(m):
    """(row, col) pairs of a reference SparseBoolMatrix or a CsrMatrix."""
    indptr = np.asarray(m.indptr, dtype=np.int64)
    indices = np.asarray(m.indices, dtype=np.int64)
    rows = np.repeat(np.arange(indptr.size - 1, dtype=np.int64), np.diff(indptr))
    return rows, indices


@dataclass
class Automaton:
    """Host mirror of rpq.query_compiler.TwoNfa (query_compiler.py:222-254)."""

    nstates: int
    transitions: dict
    starts: CsrMatrix
    finals: CsrMatrix
    alphabet: frozenset = field(default_factory=frozenset)
    label_names: dict = field(default_factory=dict)

    @property
    def start_set(self):
        return set(np.asarray(self.starts.indices).tolist())

    @property
    def final_set(self):
        return set(np.asarray(self.finals.indices).tolist())

    @classmethod
    def build(cls, nstates, transitions, starts, finals, label_names=None, alphabet=None):
        """transitions: {(label_index, inverted): [(q, q2), ...]}."""
        mats = {
            (int(k[0]), bool(k[1])): CsrMatrix.from_pairs(nstates, nstates, pairs)
            for k, pairs in transitions.items()
        }
        return cls(
            nstates=int(nstates),
            transitions=mats,
            starts=CsrMatrix.from_pairs(1, nstates, [(0, s) for s in starts]),
            finals=CsrMatrix.from_pairs(1, nstates, [(0, f) for f in finals]),
            alphabet=frozenset(mats) if alphabet is None else frozenset(
                (int(a), bool(b)) for a, b in alphabet),
            label_names=dict(label_names or {}),
        )

    @classmethod
    def from_json(cls, d):
        """Fixture format written by tests/golden/make_golden.py."""
        trans = {(int(t[0]), bool(t[1])): [tuple(p) for p in t[2]] for t in d["transitions"]}
        return cls.build(d["nstates"], trans, d["starts"], d["finals"],
                         {int(k): v for k, v in d.get("label_names", {}).items()},
                         alphabet=[tuple(a) for a in d["alphabet"]] if "alphabet" in d else None)

    def to_json(self):
        return {
            "nstates": self.nstates,
            "transitions": [[k[0], k[1], [list(p) for p in m.pairs()]]
                            for k, m in sorted(self.transitions.items())],
            "alphabet": sorted([list(a) for a in self.alphabet]),
            "starts": sorted(self.start_set),
            "finals": sorted(self.final_set),
            "label_names": {str(k): v for k, v in self.label_names.items()},
        }


def reverse(n):
    """Automaton of the reversed language (query_compiler.py:488-502):
    transposed transitions with every symbol's direction flipped, start and
    final sets swapped.  Accepts a reference TwoNfa or an Automaton."""
    trans = {}
    for (idx, inverted), m in n.transitions.items():
        rows, cols = _matrix_pairs(m)
        trans[(idx, not inverted)] = list(zip(cols.tolist(), rows.tolist()))
    return Automaton.build(n.nstates, trans, sorted(n.final_set), sorted(n.start_set),
                           dict(getattr(n, "label_names", {}) or {}))


class TransitionTable:
    """Flat (src, label, inverted, dst) arrays of the usable transitions."""

    __slots__ = ("nstates", "t_src", "t_label", "t_inv", "t_dst", "starts", "finals", "labels",
                 "key")

    def __init__(self, nstates, t_src, t_label, t_inv, t_dst, starts, finals):
        self.nstates = int(nstates)
        self.t_src = np.ascontiguousarray(t_src, dtype=np.int32)
        self.t_label = np.ascontiguousarray(t_label, dtype=np.int32)
        self.t_inv = np.ascontiguousarray(t_inv, dtype=np.uint8)
        self.t_dst = np.ascontiguousarray(t_dst, dtype=np.int32)
        self.starts = np.ascontiguousarray(starts, dtype=np.int32)
        self.finals = np.ascontiguousarray(finals, dtype=np.int32)
        self.labels = sorted(set(self.t_label.tolist()))
        h = hashlib.sha1()
        for a in (self.t_src, self.t_label, self.t_inv, self.t_dst, self.starts, self.finals):
            h.update(a.tobytes())
            h.update(b"|")
        h.update(str(self.nstates).encode())
        self.key = h.hexdigest()

    @property
    def ntrans(self):
        return int(self.t_src.size)


def transition_table(n, num_labels):
    """The usable symbols of ``n`` as a flat table, mirroring _label_pairs
    (engine.py:92-103) and _seed / _project_finals (:106-114)."""
    t_src, t_label, t_inv, t_dst = [], [], [], []
    for idx, inverted in sorted(n.alphabet):
        if not 0 <= idx < num_labels:  # g.has_label_index(idx), engine.py:100
            continue
        m = n.transitions[(idx, inverted)]
        rows, cols = _matrix_pairs(m)
        t_src.extend(rows.tolist())
        t_dst.extend(cols.tolist())
        t_label.extend([idx] * rows.size)
        t_inv.extend([1 if inverted else 0] * rows.size)
    return TransitionTable(n.nstates, t_src, t_label, t_inv, t_dst, sorted(n.start_set),
                           sorted(n.final_set))
