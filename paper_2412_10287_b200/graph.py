"""Graph residency: host-side labelled graphs and their device images.

The engine accepts the reference's own ``LabeledGraph``
(/root/reference/pkg/src/rpq/graph_store.py:28-105) duck-typed: it reads
``num_vertices``, ``num_labels``, ``has_label_index(l)`` and, per label the
query uses, ``forward[l].indptr/.indices`` and ``backward[l].indptr/.indices``
(the reference keeps both as int64 CSR, sparse_bool.py:51-59, with
``backward[l] = transpose(forward[l])``, graph_store.py:52).

``LabeledGraph`` below is a host type with the same attributes for callers who
do not have the reference package (the bench and the GPU tests): built from
per-label CSR arrays or from an edge list, with the per-label CSR materialised
lazily (a 2,000-label, 90M-vertex graph cannot hold dense row pointers for every
label: SURVEY.md §8(b)).

``DeviceGraph`` owns the ``rpq_graph`` handle: labels are uploaded on first use
by a query (the reference excludes graph loading from query time,
cli.py:98-107) and stay resident.  ``device_graph(g)`` caches one image per
host graph object.
"""

import ctypes
import threading
import weakref

import numpy as np

from . import _lib


class CsrMatrix:
    """Minimal immutable Boolean CSR (the attributes SparseBoolMatrix exposes)."""

    __slots__ = ("nrows", "ncols", "indptr", "indices")

    def __init__(self, nrows, ncols, indptr, indices):
        self.nrows = int(nrows)
        self.ncols = int(ncols)
        self.indptr = np.ascontiguousarray(indptr)
        self.indices = np.ascontiguousarray(indices)
        if self.indptr.shape != (self.nrows + 1,):
            raise ValueError("indptr must have nrows + 1 entries")

    @classmethod
    def from_pairs(cls, nrows, ncols, pairs):
        pairs = sorted(set((int(r), int(c)) for r, c in pairs))
        for r, c in pairs:
            if not (0 <= r < nrows and 0 <= c < ncols):
                raise ValueError(f"position out of bounds for {nrows}x{ncols} matrix")
        indptr = np.zeros(nrows + 1, dtype=np.int64)
        for r, _ in pairs:
            indptr[r + 1] += 1
        np.cumsum(indptr, out=indptr)
        indices = np.array([c for _, c in pairs], dtype=np.int64)
        return cls(nrows, ncols, indptr, indices)

    @property
    def nnz(self):
        return int(self.indices.size)

    @property
    def shape(self):
        return (self.nrows, self.ncols)

    def pairs(self):
        rows = np.repeat(np.arange(self.nrows, dtype=np.int64), np.diff(self.indptr))
        return list(zip(rows.tolist(), self.indices.tolist()))

    def transpose(self):
        rows = np.repeat(np.arange(self.nrows, dtype=np.int64), np.diff(self.indptr))
        cols = np.asarray(self.indices, dtype=np.int64)
        order = np.lexsort((rows, cols))
        indptr = np.zeros(self.ncols + 1, dtype=np.int64)
        np.add.at(indptr, cols + 1, 1)
        np.cumsum(indptr, out=indptr)
        return CsrMatrix(self.ncols, self.nrows, indptr, rows[order])


class _LazyLabels:
    """Sequence of per-label CsrMatrix built on first access."""

    def __init__(self, n, build):
        self._n = n
        self._build = build
        self._cache = {}
        self._lock = threading.Lock()

    def __len__(self):
        return self._n

    def __getitem__(self, label):
        if not 0 <= label < self._n:
            raise IndexError(label)
        m = self._cache.get(label)
        if m is None:
            with self._lock:
                m = self._cache.get(label)
                if m is None:
                    m = self._build(label)
                    self._cache[label] = m
        return m

    def __iter__(self):
        return (self[i] for i in range(self._n))


class LabeledGraph:
    """Host graph with the reference LabeledGraph's query-side attributes."""

    def __init__(self, num_vertices, labels, forward, backward=None, vertices=None):
        self._nv = int(num_vertices)
        self.labels = list(labels)
        self.label_ids = {name: i for i, name in enumerate(self.labels)}
        self.forward = forward
        self.backward = backward if backward is not None else [m.transpose() for m in forward]
        self._vertices = vertices

    @classmethod
    def from_edges(cls, num_vertices, labels, edges):
        """edges: iterable of (src, label_index, dst) with dense indices."""
        nl = len(labels)
        per = [[] for _ in range(nl)]
        for u, l, v in edges:
            per[l].append((u, v))
        fwd = [CsrMatrix.from_pairs(num_vertices, num_vertices, p) for p in per]
        return cls(num_vertices, labels, fwd)

    @classmethod
    def from_coo(cls, num_vertices, labels, src, dst, lab):
        """Edge list (int32 arrays) -> lazily built canonical per-label CSR
        (dedup per (src, label, dst), rows sorted: graph_store.py:161-176)."""
        src = np.ascontiguousarray(src, dtype=np.int32)
        dst = np.ascontiguousarray(dst, dtype=np.int32)
        lab = np.ascontiguousarray(lab, dtype=np.int32)
        nv = int(num_vertices)
        ne = int(src.size)
        lib = _lib.datagen()

        def build(label, transpose):
            cap = lib.rpqgen_label_count(ne, _lib.ptr(lab, ctypes.c_int32), label)
            indptr = np.empty(nv + 1, dtype=np.int64)
            indices = np.empty(max(cap, 1), dtype=np.int64)
            nnz = lib.rpqgen_label_csr(nv, ne, _lib.ptr(src, ctypes.c_int32),
                                       _lib.ptr(dst, ctypes.c_int32),
                                       _lib.ptr(lab, ctypes.c_int32), label, int(transpose),
                                       _lib.ptr(indptr, ctypes.c_int64),
                                       _lib.ptr(indices, ctypes.c_int64))
            if nnz < 0:
                raise MemoryError("label CSR build failed")
            return CsrMatrix(nv, nv, indptr, indices[:nnz].copy())

        g = cls(nv, labels, _LazyLabels(len(labels), lambda l: build(l, False)),
                _LazyLabels(len(labels), lambda l: build(l, True)))
        g._coo = (src, dst, lab)
        return g

    @property
    def num_vertices(self):
        return self._nv

    @property
    def num_labels(self):
        return len(self.labels)

    @property
    def vertices(self):
        if self._vertices is None:
            self._vertices = [str(i) for i in range(self._nv)]
        return self._vertices

    def has_label_index(self, index):
        return 0 <= index < len(self.labels)

    def adjacency(self, label, inverted=False):
        if not self.has_label_index(label):
            raise ValueError(f"unknown label index {label}")
        return self.backward[label] if inverted else self.forward[label]

    def vertex_index(self, name):
        return int(name) if self._vertices is None else self._vertices.index(name)

    def __repr__(self):
        return f"LabeledGraph(|V|={self._nv}, |L|={self.num_labels})"


# ---------------------------------------------------------------------------
# device image
# ---------------------------------------------------------------------------


def _raise_status(rc, what):
    from .engine import raise_for_status

    raise_for_status(rc, what)


class DeviceGraph:
    """Device-resident image of a host graph (``rpq_graph`` handle)."""

    def __init__(self, host_graph, device=0, ingest="auto"):
        """ingest: "csr" uploads the host's per-label CSR (forward/backward);
        "coo" uploads the edge list once and builds each label's CSR on the
        device when a query first needs it; "auto" uses "coo" when the host
        graph was built from an edge list (LabeledGraph.from_coo)."""
        try:  # weak, so the cache below does not keep host graphs alive
            self._host = weakref.ref(host_graph)
        except TypeError:
            self._host = lambda: host_graph
        self.device = int(device)
        self.num_vertices = int(host_graph.num_vertices)
        self.num_labels = int(host_graph.num_labels)
        coo = getattr(host_graph, "_coo", None)
        self.ingest = "coo" if ingest == "coo" or (ingest == "auto" and coo is not None) else "csr"
        lib = _lib.engine()
        handle = ctypes.c_void_p()
        if self.ingest == "coo":
            if coo is None:
                raise ValueError("ingest='coo' needs a graph built from an edge list")
            src, dst, lab = coo
            rc = lib.rpq_graph_create_coo(self.num_vertices, self.num_labels, int(src.size),
                                          _lib.ptr(src, ctypes.c_int32), _lib.ptr(dst, ctypes.c_int32),
                                          _lib.ptr(lab, ctypes.c_int32), self.device,
                                          ctypes.byref(handle))
        else:
            rc = lib.rpq_graph_create(self.num_vertices, self.num_labels, self.device,
                                      ctypes.byref(handle))
        if rc:
            _raise_status(rc, "rpq_graph_create")
        self.handle = handle
        self._resident = set()  # labels known to be resident (they stay resident)
        self._lock = threading.Lock()
        self._queries = {}
        self._finalizer = weakref.finalize(self, DeviceGraph._release, handle.value, self._queries)

    @property
    def host(self):
        return self._host()

    @staticmethod
    def _release(handle, queries):
        lib = _lib.engine()
        for pool in queries.values():
            for q in pool:
                lib.rpq_query_destroy(q)
        queries.clear()
        lib.rpq_graph_destroy(handle)

    def close(self):
        self._finalizer()

    def resident(self, label):
        return bool(_lib.engine().rpq_graph_label_resident(self.handle, label))

    def ensure_labels(self, labels):
        """Upload every listed label (forward + backward CSR) not yet resident."""
        if self._resident.issuperset(labels):  # the per-query fast path: no C call
            return
        lib = _lib.engine()
        for label in labels:
            if lib.rpq_graph_label_resident(self.handle, label):
                self._resident.add(label)
                continue
            if self.ingest == "coo":
                rc = lib.rpq_graph_materialize_label(self.handle, label)
                if rc:
                    _raise_status(rc, f"device build of label {label}")
                self._resident.add(label)
                continue
            host = self.host
            if host is None:
                raise RuntimeError("host graph of this device image was released")
            fwd = host.forward[label]
            bwd = host.backward[label]
            fp, fi = np.ascontiguousarray(fwd.indptr), np.ascontiguousarray(fwd.indices)
            bp, bi = np.ascontiguousarray(bwd.indptr), np.ascontiguousarray(bwd.indices)
            if fp.dtype == np.int32 and fi.dtype == np.int32 and bp.dtype == np.int32 \
                    and bi.dtype == np.int32:
                rc = lib.rpq_graph_set_label_i32(
                    self.handle, label, fi.size, _lib.ptr(fp, ctypes.c_int32),
                    _lib.ptr(fi, ctypes.c_int32), bi.size, _lib.ptr(bp, ctypes.c_int32),
                    _lib.ptr(bi, ctypes.c_int32))
            else:
                fp, fi, bp, bi = (np.ascontiguousarray(a, dtype=np.int64) for a in (fp, fi, bp, bi))
                rc = lib.rpq_graph_set_label(
                    self.handle, label, fi.size, _lib.ptr(fp, ctypes.c_int64),
                    _lib.ptr(fi, ctypes.c_int64), bi.size, _lib.ptr(bp, ctypes.c_int64),
                    _lib.ptr(bi, ctypes.c_int64))
            if rc:
                _raise_status(rc, f"upload of label {label}")
            self._resident.add(label)

    def label_csr(self, label, transpose=False):
        """(rowptr uint32[|V|+1], col int32[nnz]) of a resident label, copied back."""
        lib = _lib.engine()
        nnz = ctypes.c_int64()
        rc = lib.rpq_graph_copy_label(self.handle, label, int(transpose), None, None, 0, ctypes.byref(nnz))
        if rc:
            _raise_status(rc, "rpq_graph_copy_label")
        rowptr = np.empty(self.num_vertices + 1, dtype=np.uint32)
        col = np.empty(max(nnz.value, 1), dtype=np.int32)
        rc = lib.rpq_graph_copy_label(self.handle, label, int(transpose), _lib.ptr(rowptr, ctypes.c_uint32),
                                      _lib.ptr(col, ctypes.c_int32), col.size, ctypes.byref(nnz))
        if rc:
            _raise_status(rc, "rpq_graph_copy_label")
        return rowptr, col[: nnz.value]

    @property
    def device_bytes(self):
        return int(_lib.engine().rpq_graph_device_bytes(self.handle))

    # -- query objects (device workspaces), pooled per transition table -------
    def acquire_query(self, table, private=False):
        """A query handle for ``table``: from the per-table pool, or (private)
        a fresh one the caller may retune and must give back with
        ``destroy_query`` -- never to the pool, so that eval_ssr never
        inherits a PreparedQuery's tuning."""
        key = table.key
        if not private:
            with self._lock:
                pool = self._queries.setdefault(key, [])
                if pool:
                    return pool.pop()
        lib = _lib.engine()
        h = ctypes.c_void_p()
        rc = lib.rpq_query_create(
            self.handle, table.nstates, table.ntrans, _lib.ptr(table.t_src, ctypes.c_int32),
            _lib.ptr(table.t_label, ctypes.c_int32), _lib.ptr(table.t_inv, ctypes.c_uint8),
            _lib.ptr(table.t_dst, ctypes.c_int32), table.starts.size,
            _lib.ptr(table.starts, ctypes.c_int32), table.finals.size,
            _lib.ptr(table.finals, ctypes.c_int32), ctypes.byref(h))
        if rc:
            _raise_status(rc, "rpq_query_create")
        return h.value

    def release_query(self, table, q):
        with self._lock:
            self._queries.setdefault(table.key, []).append(q)

    def destroy_query(self, q):
        if q:
            _lib.engine().rpq_query_destroy(q)


_DEVICE_GRAPHS = weakref.WeakKeyDictionary()
_DEVICE_GRAPHS_BY_ID = {}
_CACHE_LOCK = threading.Lock()


def device_graph(g, device=0):
    """Cached DeviceGraph for host graph ``g`` (keyed by object identity)."""
    if isinstance(g, DeviceGraph):
        return g
    key = (id(g), int(device))
    with _CACHE_LOCK:
        try:
            per = _DEVICE_GRAPHS.get(g)
        except TypeError:  # not weak-referenceable
            per = None
            hit = _DEVICE_GRAPHS_BY_ID.get(key)
            if hit is not None and hit.host is g:
                return hit
        if per is not None and int(device) in per:
            return per[int(device)]
        dg = DeviceGraph(g, device)
        try:
            _DEVICE_GRAPHS.setdefault(g, {})[int(device)] = dg
        except TypeError:
            _DEVICE_GRAPHS_BY_ID[key] = dg
        return dg
