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


def desk_bench():
    """The reference's desk-scale benchmark (test_acceptance.py:238-335):
    (golden record, graph arrays) from tests/golden/desk_bench.json.gz and
    desk_graph.npz (written by make_golden.py desk)."""
    import os

    from conftest import GOLDEN, load_golden

    rec = load_golden("desk_bench.json.gz")
    z = np.load(os.path.join(GOLDEN, "desk_graph.npz"))
    nl = len(rec["labels"])
    csr = [(z[f"indptr_{l}"].astype(np.int64), z[f"indices_{l}"].astype(np.int64)) for l in range(nl)]
    return rec, csr


def desk_host_graph(rec, csr):
    nv = rec["nv"]
    return LabeledGraph(nv, rec["labels"], [CsrMatrix(nv, nv, ip, ix) for ip, ix in csr])


def desk_oracle_graph(rec, csr):
    from oracle import OracleGraph

    src, dst, lab = [], [], []
    for l, (ip, ix) in enumerate(csr):
        src.append(np.repeat(np.arange(rec["nv"], dtype=np.int32), np.diff(ip)))
        dst.append(ix.astype(np.int32))
        lab.append(np.full(ix.size, l, dtype=np.int32))
    return OracleGraph(rec["nv"], len(csr), np.concatenate(src), np.concatenate(dst), np.concatenate(lab))


def answer_digest(reach):
    """sha256 of the comma-joined sorted answer ids (test_acceptance.py:338-351's format)."""
    import hashlib

    return hashlib.sha256(",".join(str(v) for v in np.flatnonzero(reach).tolist()).encode()).hexdigest()


def reach_sha256(reach):
    """sha256 of the little-endian packed answer bitmap (make_golden.reach_digest)."""
    import hashlib

    return hashlib.sha256(np.packbits(np.asarray(reach, dtype=np.uint8), bitorder="little").tobytes()).hexdigest()
