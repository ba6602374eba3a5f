"""Test-only pieces for the vertex-partitioned evaluator: a numpy step over a
rank's local problem (so the partition / exchange / termination logic runs on
CPU under gloo) and the bitmap packing it needs."""

import numpy as np

from paper_2412_10287_b200.automaton import transition_table


def pack_rows(b, row_words):
    """bool [Q, nv] -> int32 [Q, row_words] (bit v%32 of word v/32)."""
    q, nv = b.shape
    out = np.zeros((q, row_words * 32), dtype=bool)
    out[:, :nv] = b
    return np.packbits(out, axis=1, bitorder="little").view(np.uint32).view(np.int32)


def unpack_rows(w, nv):
    return np.unpackbits(np.ascontiguousarray(w).view(np.uint8), axis=1, bitorder="little")[:, :nv].astype(bool)


class CpuStep:
    """next = step(M) <not P>, P |= next on CPU torch tensors (tests only)."""

    def __init__(self, lg, ln, nv):
        self.nv = nv
        self.row_words = ((nv + 31) // 32 + 3) // 4 * 4
        t = transition_table(ln, lg.num_labels)
        self.trans = list(zip(t.t_src.tolist(), t.t_label.tolist(), t.t_inv.tolist(), t.t_dst.tolist()))
        self.adj = {(l, inv): lg.adjacency(l, bool(inv)) for _, l, inv, _ in self.trans}

    def __call__(self, m, p, out, stream):
        import torch

        M = unpack_rows(m.numpy(), self.nv)
        P = unpack_rows(p.numpy(), self.nv)
        N = np.zeros_like(M)
        for s, l, inv, d in self.trans:
            a = self.adj[(l, inv)]
            indptr = np.asarray(a.indptr)
            for r in np.flatnonzero(M[s]):
                N[d, np.asarray(a.indices[indptr[r]:indptr[r + 1]])] = True
        N &= ~P
        P |= N
        out.copy_(torch.from_numpy(pack_rows(N, self.row_words)))
        p.copy_(torch.from_numpy(pack_rows(P, self.row_words)))
