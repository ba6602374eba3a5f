"""Seeded synthetic inputs for the five BASELINE.json configurations.

The reference benchmarks on Wikidata / Yago / RPQBench,
none of which is available here; these generators stand in with the shapes,
sizes and value distributions BASELINE.json names.  All
draws are counter-based (csrc/datagen.c), so the arrays are a pure function of
the config and identical across machines and thread counts; both the CUDA
engine and the CPU oracle consume the same arrays.

Label names follow the Zipf rank: rank 1 is ``a`` (``a1`` for cfg5), rank 2
``b`` (``a2``), ...; label index = rank - 1.
"""

import ctypes
import string
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .graph import LabeledGraph

RMAT_ABC = (0.57, 0.19, 0.19)


def rank_names(nl, style="letters"):
    if style == "a_index":
        return [f"a{k + 1}" for k in range(nl)]
    letters = string.ascii_lowercase
    return [letters[k] if k < 26 else f"l{k}" for k in range(nl)]


CHAIN16 = " ".join(f"(a{2 * i + 1} a{2 * i + 2}*)" for i in range(8))
CHAIN16_TWOWAY = " ".join(f"(a{2 * i + 1} ^a{2 * i + 2}*)" for i in range(8))
# the two-way variant on even labels in both directions: 25 states unminimized
CHAIN16_BOTHWAY = " ".join(f"(a{2 * i + 1} (a{2 * i + 2}|^a{2 * i + 2})*)" for i in range(8))

CONFIGS = {
    # cfg1: Erdos-Renyi 10k / 100k, 4 uniform labels, query a b*, source 0
    "cfg1": dict(kind="er", nv=10_000, ne=100_000, nl=4, seed=1, names="letters",
                 queries=["a b*"], sources="zero"),
    # cfg2: R-MAT scale 20, edge factor 16, 16 Zipf(1.0) labels, a ^b* c,
    # source = highest total out-degree vertex
    "cfg2": dict(kind="rmat", scale=20, ef=16, nl=16, zipf=1.0, seed=2, names="letters",
                 queries=["a ^b* c"], sources="max_out_degree"),
    # cfg3: R-MAT scale 24, 64 labels, ^a (b|c)* d, uniform sources with out-degree >= 1
    "cfg3": dict(kind="rmat", scale=24, ef=16, nl=64, zipf=1.0, seed=3, names="letters",
                 queries=["^a (b|c)* d"], sources="uniform_outdeg", nsources=8),
    # cfg4: Chung-Lu 90M / 1.2B, exponent 2.1, 2,000 Zipf(1.1) labels, 4 templates x 32 sources
    "cfg4": dict(kind="chunglu", nv=90_000_000, ne=1_200_000_000, gamma=2.1, nl=2000, zipf=1.1,
                 seed=4, names="letters", queries=["a*", "a+ b", "(a|b|c|d)*", "a ^b c*"],
                 sources="uniform_outdeg", nsources=32),
    # cfg5: R-MAT scale 22, 32 labels, 8-group chain (+ two-way variant), 1,024 sources
    "cfg5": dict(kind="rmat", scale=22, ef=16, nl=32, zipf=1.0, seed=5, names="a_index",
                 queries=[CHAIN16, CHAIN16_TWOWAY, CHAIN16_BOTHWAY], sources="uniform_outdeg", nsources=1024),
}


@dataclass
class SyntheticGraph:
    name: str
    nv: int
    label_names: list
    src: np.ndarray
    dst: np.ndarray
    lab: np.ndarray
    seed: int
    _graph: object = field(default=None, repr=False)

    @property
    def ne(self):
        return int(self.src.size)

    @property
    def nl(self):
        return len(self.label_names)

    def labeled_graph(self):
        """Host LabeledGraph (per-label int64 CSR, built lazily per label)."""
        if self._graph is None:
            self._graph = LabeledGraph.from_coo(self.nv, self.label_names, self.src, self.dst,
                                                self.lab)
        return self._graph

    def out_degree(self):
        out = np.empty(self.nv, dtype=np.int64)
        _lib.datagen().rpqgen_out_degree(self.nv, self.ne, _lib.ptr(self.src, ctypes.c_int32),
                                         _lib.ptr(out, ctypes.c_int64))
        return out

    def digest(self):
        """Order-sensitive checksum of the edge arrays (fixture pinning)."""
        import hashlib

        h = hashlib.sha256()
        for a in (self.src, self.dst, self.lab):
            h.update(np.ascontiguousarray(a).tobytes())
        return h.hexdigest()[:32]


def _alloc(n):
    return (np.empty(n, dtype=np.int32), np.empty(n, dtype=np.int32), np.empty(n, dtype=np.int32))


def gen_er(nv, ne, nl, seed, names="letters"):
    lib = _lib.datagen()
    src, dst, lab = _alloc(ne)
    n = lib.rpqgen_er(nv, ne, nl, seed, _lib.ptr(src, ctypes.c_int32),
                      _lib.ptr(dst, ctypes.c_int32), _lib.ptr(lab, ctypes.c_int32))
    if n < 0:
        raise ValueError("rpqgen_er failed")
    return SyntheticGraph("er", nv, rank_names(nl, names), src, dst, lab, seed)


def gen_rmat(scale, ef, nl, zipf, seed, names="letters", abc=RMAT_ABC):
    lib = _lib.datagen()
    m = ef << scale
    src, dst, lab = _alloc(m)
    n = lib.rpqgen_rmat(scale, m, abc[0], abc[1], abc[2], nl, zipf, seed,
                        _lib.ptr(src, ctypes.c_int32), _lib.ptr(dst, ctypes.c_int32),
                        _lib.ptr(lab, ctypes.c_int32))
    if n < 0:
        raise MemoryError("rpqgen_rmat failed")
    return SyntheticGraph("rmat", 1 << scale, rank_names(nl, names), src[:n].copy(),
                          dst[:n].copy(), lab[:n].copy(), seed)


def gen_chunglu(nv, ne, gamma, nl, zipf, seed, names="letters"):
    lib = _lib.datagen()
    src, dst, lab = _alloc(ne)
    n = lib.rpqgen_chunglu(nv, ne, gamma, nl, zipf, seed, _lib.ptr(src, ctypes.c_int32),
                           _lib.ptr(dst, ctypes.c_int32), _lib.ptr(lab, ctypes.c_int32))
    if n < 0:
        raise MemoryError("rpqgen_chunglu failed")
    return SyntheticGraph("chunglu", nv, rank_names(nl, names), src[:n], dst[:n], lab[:n], seed)


def generate(config, **overrides):
    """SyntheticGraph for a config name ("cfg1".."cfg5"); overrides e.g. scale=16."""
    c = dict(CONFIGS[config])
    c.update(overrides)
    if c["kind"] == "er":
        g = gen_er(c["nv"], c["ne"], c["nl"], c["seed"], c["names"])
    elif c["kind"] == "rmat":
        g = gen_rmat(c["scale"], c["ef"], c["nl"], c["zipf"], c["seed"], c["names"])
    else:
        g = gen_chunglu(c["nv"], c["ne"], c["gamma"], c["nl"], c["zipf"], c["seed"], c["names"])
    g.name = config
    return g


def pick_sources(g, config, count=None, **overrides):
    """Query sources of a config:
    zero -> [0]; max_out_degree -> argmax total out-degree (ties: lowest id);
    uniform_outdeg -> `count` draws, uniform over vertices with out-degree >= 1,
    from the counter-based generator (seed + 100)."""
    c = dict(CONFIGS[config])
    c.update(overrides)
    kind = c["sources"]
    if kind == "zero":
        return [0]
    deg = g.out_degree()
    if kind == "max_out_degree":
        return [int(np.argmax(deg))]
    cand = np.flatnonzero(deg > 0)
    n = count if count is not None else c.get("nsources", 1)
    lib = _lib.datagen()
    out = []
    for j in range(n):
        r = lib.rpqgen_draw(c["seed"] + 100, 7, j)
        out.append(int(cand[(r >> 32) * cand.size >> 32]))
    return out
