"""ctypes wrapper of the CPU oracle (rpq_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs -- never by the product
package.  See rpq_oracle.c for what each entry point restates (file:line of
/root/reference/pkg/src/rpq) and tests/test_oracle_golden.py for the pin
against the reference's own outputs.
"""

import ctypes
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "liboracle.so")
MAX_LEVELS = 4096

ALGORITHM_CODES = {"masked": 0, "no_mask": 1, "hybrid": 2}


class OStats(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int32),
        ("levels", ctypes.c_int32),
        ("te", ctypes.c_int64),
        ("x", ctypes.c_int64),
        ("pairs", ctypes.c_int64),
        ("reach", ctypes.c_int64),
        ("seconds", ctypes.c_double),
        ("level_new", ctypes.c_int64 * MAX_LEVELS),
    ]

    def to_dict(self):
        return {
            "iterations": self.iterations,
            "levels": self.levels,
            "te": self.te,
            "x": self.x,
            "pairs": self.pairs,
            "reach": self.reach,
            "seconds": self.seconds,
            "level_new": list(self.level_new[: min(self.levels, MAX_LEVELS)]),
        }


_lib = None
_lock = threading.Lock()

_P32 = ctypes.POINTER(ctypes.c_int32)
_P64 = ctypes.POINTER(ctypes.c_int64)
_PU8 = ctypes.POINTER(ctypes.c_uint8)


def build():
    src = os.path.join(HERE, "rpq_oracle.c")
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return SO


def lib():
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                build()
                L = ctypes.CDLL(SO)
                L.oracle_graph_create.restype = ctypes.c_void_p
                L.oracle_graph_create.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int64,
                                                  _P32, _P32, _P32]
                L.oracle_graph_destroy.argtypes = [ctypes.c_void_p]
                L.oracle_graph_prepare.restype = ctypes.c_int64
                L.oracle_graph_prepare.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32]
                L.oracle_graph_slot.restype = ctypes.c_int64
                L.oracle_graph_slot.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                                _P64, _P32]
                common = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, _P32, _P32, _P32, _P32,
                          ctypes.c_int32, _P32, ctypes.c_int32, _P32, ctypes.c_int32]
                L.oracle_bfs.restype = ctypes.c_int
                L.oracle_bfs.argtypes = common + [_PU8, ctypes.POINTER(OStats)]
                L.oracle_port.restype = ctypes.c_int
                L.oracle_port.argtypes = common + [ctypes.c_int32, ctypes.c_double,
                                                   ctypes.c_double, _PU8, ctypes.POINTER(OStats)]
                _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


class OracleGraph:
    """Edge list (src, label, dst) with lazily built per-label CSR (C side)."""

    def __init__(self, nv, nl, src, dst, lab):
        self.nv = int(nv)
        self.nl = int(nl)
        self.src = np.ascontiguousarray(src, dtype=np.int32)
        self.dst = np.ascontiguousarray(dst, dtype=np.int32)
        self.lab = np.ascontiguousarray(lab, dtype=np.int32)
        self.h = lib().oracle_graph_create(self.nv, self.nl, self.src.size,
                                           _p(self.src, ctypes.c_int32),
                                           _p(self.dst, ctypes.c_int32),
                                           _p(self.lab, ctypes.c_int32))

    @classmethod
    def from_label_pairs(cls, nv, per_label_pairs):
        """per_label_pairs: list over labels of [(u, v), ...]."""
        src, dst, lab = [], [], []
        for l, pairs in enumerate(per_label_pairs):
            for u, v in pairs:
                src.append(u)
                dst.append(v)
                lab.append(l)
        return cls(nv, len(per_label_pairs), np.array(src, dtype=np.int32),
                   np.array(dst, dtype=np.int32), np.array(lab, dtype=np.int32))

    def prepare(self, label, inverted):
        return int(lib().oracle_graph_prepare(self.h, label, int(inverted)))

    def slot_csr(self, label, inverted):
        nnz = self.prepare(label, inverted)
        indptr = np.empty(self.nv + 1, dtype=np.int64)
        indices = np.empty(max(nnz, 1), dtype=np.int32)
        lib().oracle_graph_slot(self.h, label, int(inverted), _p(indptr, ctypes.c_int64),
                                _p(indices, ctypes.c_int32))
        return indptr, indices[:nnz]

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.oracle_graph_destroy(self.h)
            self.h = None


class OracleQuery:
    """Transition triples of an automaton, read the way the reference engine
    reads it: sorted(alphabet), skipping label indices >= num_labels
    (engine.py:92-103).  `automaton` is a dict in the fixture format:
    {"nstates", "transitions": [[idx, inv, [[q, q2], ...]], ...], "alphabet",
     "starts", "finals"}."""

    def __init__(self, automaton, num_labels):
        a = automaton
        mats = {(int(t[0]), bool(t[1])): t[2] for t in a["transitions"]}
        alphabet = sorted((int(x[0]), bool(x[1])) for x in a.get("alphabet", list(mats)))
        src, lab, inv, dst = [], [], [], []
        for idx, inverted in alphabet:
            if not 0 <= idx < num_labels:
                continue
            for q, q2 in mats[(idx, inverted)]:
                src.append(q)
                lab.append(idx)
                inv.append(int(inverted))
                dst.append(q2)
        self.nstates = int(a["nstates"])
        self.t_src = np.array(src, dtype=np.int32)
        self.t_label = np.array(lab, dtype=np.int32)
        self.t_inv = np.array(inv, dtype=np.int32)
        self.t_dst = np.array(dst, dtype=np.int32)
        self.starts = np.array(sorted(set(a["starts"])), dtype=np.int32)
        self.finals = np.array(sorted(set(a["finals"])), dtype=np.int32)
        self.slots = sorted(set(zip(lab, inv)))

    def _args(self, og):
        return (og.h, self.nstates, self.t_src.size, _p(self.t_src, ctypes.c_int32),
                _p(self.t_label, ctypes.c_int32), _p(self.t_inv, ctypes.c_int32),
                _p(self.t_dst, ctypes.c_int32), self.starts.size, _p(self.starts, ctypes.c_int32),
                self.finals.size, _p(self.finals, ctypes.c_int32))

    def prepare(self, og):
        for l, i in self.slots:
            og.prepare(l, i)


def oracle_bfs(og, oq, source):
    """(reach uint8[|V|], stats) by level-synchronous product BFS."""
    reach = np.zeros(og.nv, dtype=np.uint8)
    st = OStats()
    rc = lib().oracle_bfs(*oq._args(og), int(source), _p(reach, ctypes.c_uint8),
                          ctypes.byref(st))
    if rc == 2:
        raise IndexError(f"vertex index {source} out of range")
    if rc:
        raise ValueError(f"oracle_bfs failed ({rc})")
    return reach, st.to_dict()


def oracle_port(og, oq, source, algorithm="hybrid", threshold=100.0, timeout=-1.0):
    """(reach, stats) by the reference's own masked / no_mask / hybrid loops
    on sorted key sets.  Raises TimeoutError on timeout."""
    reach = np.zeros(og.nv, dtype=np.uint8)
    st = OStats()
    rc = lib().oracle_port(*oq._args(og), int(source), ALGORITHM_CODES[algorithm],
                           float(threshold), float(timeout), _p(reach, ctypes.c_uint8),
                           ctypes.byref(st))
    if rc == 2:
        raise IndexError(f"vertex index {source} out of range")
    if rc == 3:
        raise TimeoutError(st.iterations)
    if rc:
        raise ValueError(f"oracle_port failed ({rc})")
    return reach, st.to_dict()
