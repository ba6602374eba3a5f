"""Turn golden fixture records into the objects each side consumes."""

import base64

import numpy as np

from paper_2412_10287_b200 import Automaton, LabeledGraph
from paper_2412_10287_b200.graph import CsrMatrix


def host_graph(gj):
    """Package LabeledGraph (per-label int64 CSR, like the reference's)."""
    nv = gj["nv"]
    fwd = [CsrMatrix.from_pairs(nv, nv, [tuple(p) for p in pairs]) for pairs in gj["edges"]]
    return LabeledGraph(nv, gj["labels"], fwd, vertices=gj.get("vertices"))


def oracle_graph(gj):
    from oracle import OracleGraph

    return OracleGraph.from_label_pairs(gj["nv"], [[tuple(p) for p in e] for e in gj["edges"]])


def automaton(nj):
    return Automaton.from_json(nj)


def expected_reach(rec, nv):
    out = np.zeros(nv, dtype=np.uint8)
    out[rec["expected"]] = 1
    return out


def unpack_bits(b64, nv):
    raw = np.frombuffer(base64.b64decode(b64), dtype=np.uint8)
    return np.unpackbits(raw, bitorder="little")[:nv].astype(np.uint8)
