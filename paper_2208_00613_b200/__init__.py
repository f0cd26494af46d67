"""B200-native IMM hot path with HBMax's compress-to-compute RRR storage.

A drop-in for the reference's Python module ``immx`` (proj/python/immx/__init__.py,
proj/bindings/module.cpp:56-250): the same 26 names with the same arguments, return shapes
and exception classes.  Every call goes through the C-ABI of ``include/immx_b200.h``
(``libimmx_b200.so``); sampling, histograms, encoding, decoding and greedy selection run as
sm_100a kernels.  Host-side pieces are the ones the reference also keeps scalar: graph
ingestion, theta arithmetic, characterization and the Huffman tree.

Results are bit-identical to the reference for the same graph, seed and parameters: the
per-sample random stream of proj/include/immx/rng.hpp is reproduced on the device.
"""
from __future__ import annotations

import ctypes as C
import resource
import time

import numpy as np

from . import _capi
from ._capi import arr, check, lib, ptr

__version__ = "0.1.0"

__all__ = [
    "BitmapCollection", "EncodedRrr", "Graph", "HuffmanCodebook", "assign_weights", "build_codebook",
    "choose_encoding", "decode_find", "density", "encode_bitmap", "encode_rrr", "estimate_theta",
    "load_edge_list", "load_edge_list_text", "load_graph_cache", "merged_argmax", "run", "sample_block",
    "sample_rrr", "save_graph_cache", "select_raw", "skewness", "table_argmax", "theta_bound",
    "theta_bound_real", "transpose",
    # the C++ API's stats output (pipeline.hpp:66-71)
    "stats_to_json", "write_stats", "write_seeds",
    # B200 additions
    "Device", "default_device", "generate_rmat", "generate_er", "DeviceGraph", "Pool", "run_device",
]

# "hybrid" (builder extension): the Huffman store with n-bit bitmaps for sets above n/32
_MODE_ID = {"huffman": _capi.MODE_HUFFMAN, "bitmap": _capi.MODE_BITMAP, "raw": _capi.MODE_RAW,
            "hybrid": _capi.MODE_HYBRID}
_MODE_NAME = {v: k for k, v in _MODE_ID.items()}


# ----------------------------------------------------------------------------- device
class Device:
    """One CUDA context + stream (immx_device)."""

    def __init__(self, ordinal: int = 0, shared: bool = False):
        """shared=True: the process's shared context (immx_device_shared), which other users
        of the library in this process -- e.g. the reference module rebuilt on it
        (integration/) -- see too; otherwise an exclusive one."""
        h = C.c_void_p()
        check((lib.immx_device_shared if shared else lib.immx_device_create)(ordinal, C.byref(h)))
        self.h = h
        self.ordinal = ordinal

    @property
    def stream(self) -> int:
        return lib.immx_device_stream(self.h) or 0

    def synchronize(self):
        check(lib.immx_device_synchronize(self.h))

    @property
    def kernel_launches(self) -> int:
        return lib.immx_device_kernel_launches(self.h)

    def profile(self, enable: bool = True):
        """Bracket the hot kernels with CUDA events on the device stream."""
        check(lib.immx_device_profile(self.h, int(enable)))

    def reset_stats(self):
        check(lib.immx_device_reset_stats(self.h))

    def kernel_stats(self, kind: str):
        """-> {launches, ms, bytes}: device time and ALGORITHMIC bytes of one kernel class."""
        n, ms, b = C.c_uint64(), C.c_double(), C.c_uint64()
        check(lib.immx_device_kernel_stats(self.h, _capi.KSTAT[kind], C.byref(n), C.byref(ms), C.byref(b)))
        return {"launches": n.value, "ms": ms.value, "bytes": b.value}

    def __del__(self):
        try:
            if self.h:
                lib.immx_device_destroy(self.h)
        except Exception:
            pass


_DEFAULT = None


def default_device(ordinal: int | None = None) -> Device:
    """The process's immx_device (the C-ABI admits one live context per process)."""
    global _DEFAULT
    if _DEFAULT is None:
        _DEFAULT = Device(0 if ordinal is None else ordinal, shared=True)
    elif ordinal is not None and ordinal != _DEFAULT.ordinal:
        raise ValueError(f"the process already uses cuda:{_DEFAULT.ordinal} (one immx_device per process)")
    return _DEFAULT


# ------------------------------------------------------------------------------ graph
class Graph:
    """Host CSR graph (immx::Graph, graph.hpp:15-25)."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def from_csr(cls, n, offsets, targets, probs, original_ids=None):
        off, tgt, pr = arr(offsets, np.uint64), arr(targets, np.uint32), arr(probs, np.float64)
        ids = None if original_ids is None else arr(original_ids, np.uint64)
        h = C.c_void_p()
        check(lib.immx_hgraph_from_csr(n, tgt.size, ptr(off, C.c_uint64), ptr(tgt, C.c_uint32),
                                       ptr(pr, C.c_double), ptr(ids, C.c_uint64), C.byref(h)))
        return cls(h)

    def __del__(self):
        try:
            if self._h:
                lib.immx_hgraph_destroy(self._h)
        except Exception:
            pass

    def _info(self):
        n, m = C.c_uint64(), C.c_uint64()
        check(lib.immx_hgraph_info(self._h, C.byref(n), C.byref(m)))
        return n.value, m.value

    @property
    def n(self) -> int:
        return self._info()[0]

    @property
    def m(self) -> int:
        return self._info()[1]

    def arrays(self):
        """(offsets u64[n+1], targets u32[m], probs f64[m], original_ids u64[n]) -- copies."""
        n, m = self._info()
        o, t, p, i = C.POINTER(C.c_uint64)(), C.POINTER(C.c_uint32)(), C.POINTER(C.c_double)(), C.POINTER(C.c_uint64)()
        check(lib.immx_hgraph_view(self._h, C.byref(o), C.byref(t), C.byref(p), C.byref(i)))
        off = np.ctypeslib.as_array(o, (n + 1,)).copy()
        tgt = np.ctypeslib.as_array(t, (m,)).copy() if m else np.zeros(0, np.uint32)
        pr = np.ctypeslib.as_array(p, (m,)).copy() if m else np.zeros(0, np.float64)
        ids = np.ctypeslib.as_array(i, (n,)).copy() if n else np.zeros(0, np.uint64)
        return off, tgt, pr, ids

    @property
    def offsets(self):
        return self.arrays()[0]

    @property
    def targets(self):
        return self.arrays()[1]

    @property
    def probs(self):
        return self.arrays()[2]

    @property
    def original_ids(self):
        return self.arrays()[3]

    def out_degree(self, v: int) -> int:
        off = self.offsets
        return int(off[v + 1] - off[v])

    def __repr__(self):
        n, m = self._info()
        return f"Graph(n={n}, m={m})"


def _new_graph(fn, *args) -> Graph:
    h = C.c_void_p()
    check(fn(*args, C.byref(h)))
    return Graph(h)


def load_edge_list(path: str, directed: bool = False) -> Graph:
    return _new_graph(lib.immx_hgraph_load_edge_list, path.encode(), int(directed))


def load_edge_list_text(text: str, directed: bool = False) -> Graph:
    b = text.encode()
    return _new_graph(lib.immx_hgraph_load_edge_text, b, len(b), int(directed))


def transpose(g: Graph) -> Graph:
    return _new_graph(lib.immx_hgraph_transpose, g._h)


def _weight_model(name: str) -> int:
    if name in ("wc", "weighted-cascade"):
        return 0
    if name == "uniform":
        return 1
    raise ValueError(f"unknown weight model '{name}'")


def assign_weights(graph: Graph, model: str = "wc", p: float = 0.1) -> None:
    check(lib.immx_hgraph_assign_weights(graph._h, _weight_model(model), p))


def assign_weights_f32(graph: Graph, model: str = "wc", p: float = 0.1) -> None:
    """The BASELINE configs' weights: the reference formula rounded through float32."""
    check(lib.immx_hgraph_assign_weights_f32(graph._h, _weight_model(model), p))


def save_graph_cache(g: Graph, path: str) -> None:
    check(lib.immx_hgraph_save_cache(g._h, path.encode()))


def load_graph_cache(path: str) -> Graph:
    return _new_graph(lib.immx_hgraph_load_cache, path.encode())


def generate_rmat(scale: int, edge_factor: int, a=0.57, b=0.19, c=0.19, seed=1) -> Graph:
    return _new_graph(lib.immx_hgraph_generate_rmat, scale, edge_factor, a, b, c, seed)


def generate_er(n: int, m: int, seed: int = 0) -> Graph:
    return _new_graph(lib.immx_hgraph_generate_er, n, m, seed)


def lt_weights(g_t: Graph, seed: int = 0) -> np.ndarray:
    w = np.zeros(max(g_t.m, 1), np.float32)
    check(lib.immx_hgraph_lt_weights(g_t._h, seed, ptr(w, C.c_float)))
    return w[: g_t.m]


class DeviceGraph:
    """A graph resident in HBM (immx_graph): reverse CSR + coin thresholds."""

    def __init__(self, g: Graph, transposed: bool, device: Device | None = None, lt_weights=None):
        self.device = device or default_device()
        off, tgt, pr, _ = g.arrays()
        self.n, self.m = int(off.size - 1), int(tgt.size)
        h = C.c_void_p()
        check(lib.immx_graph_upload(self.device.h, self.n, self.m, ptr(off, C.c_uint64), ptr(tgt, C.c_uint32),
                                    ptr(pr, C.c_double), int(transposed), C.byref(h)))
        self.h = h
        if lt_weights is not None:
            w = arr(lt_weights, np.float32)
            check(lib.immx_graph_set_lt_weights(self.h, ptr(w, C.c_float)))

    @classmethod
    def from_arrays(cls, n, off, tgt, pr, transposed, device=None, weights=None, p=0.1):
        """CSR arrays (host) -> HBM.  pr: f64 per edge; or pr=None with weights="wc" / "uniform"
        (assign_weights with float32 values, applied on the device: only the CSR is copied)."""
        self = cls.__new__(cls)
        self.device = device or default_device()
        self.n, self.m = int(n), int(tgt.size)
        h = C.c_void_p()
        if pr is None:
            check(lib.immx_graph_upload_model(self.device.h, self.n, self.m, ptr(off, C.c_uint64), ptr(tgt, C.c_uint32),
                                              _weight_model(weights or "wc"), float(p), int(transposed), C.byref(h)))
        else:
            check(lib.immx_graph_upload(self.device.h, self.n, self.m, ptr(off, C.c_uint64), ptr(tgt, C.c_uint32),
                                        ptr(pr, C.c_double), int(transposed), C.byref(h)))
        self.h = h
        return self

    @classmethod
    def generate_rmat(cls, scale, edge_factor, a=0.57, b=0.19, c=0.19, seed=1, weights="wc", p=0.1, device=None):
        """R-MAT generated in HBM as the reverse CSR (identical to generate_rmat + transpose)."""
        self = cls.__new__(cls)
        self.device = device or default_device()
        h = C.c_void_p()
        check(lib.immx_graph_generate_rmat(self.device.h, scale, edge_factor, a, b, c, seed, _weight_model(weights), p,
                                           C.byref(h)))
        self.h = h
        n, m = C.c_uint64(), C.c_uint64()
        check(lib.immx_graph_info(h, C.byref(n), C.byref(m), None))
        self.n, self.m = n.value, m.value
        return self

    def download(self, probs: bool = True):
        """-> (row u64[n+1], col u32[m], prob f64[m] or None): the reverse CSR."""
        row = np.zeros(self.n + 1, np.uint64)
        col = np.zeros(max(self.m, 1), np.uint32)
        pr = np.zeros(max(self.m, 1), np.float64) if probs else None
        check(lib.immx_graph_download(self.h, ptr(row, C.c_uint64), ptr(col, C.c_uint32),
                                      None if pr is None else ptr(pr, C.c_double)))
        return row, col[: self.m], None if pr is None else pr[: self.m]

    def set_lt_weights(self, weights):
        """LT extension: per-Gt-edge float32 weights (Gt CSR order)."""
        w = arr(weights, np.float32)
        check(lib.immx_graph_set_lt_weights(self.h, ptr(w, C.c_float)))

    def set_lt_random(self, seed: int):
        """LT extension: the generator's U(0,1)-normalised weights, computed in HBM."""
        check(lib.immx_graph_set_lt_random(self.h, seed))

    @property
    def prob_mode(self) -> str:
        pm = C.c_int()
        check(lib.immx_graph_info(self.h, None, None, C.byref(pm)))
        return ["global", "row", "edge"][pm.value]

    def __del__(self):
        try:
            if self.h:
                lib.immx_graph_destroy(self.h)
        except Exception:
            pass


class Pool:
    """Device-resident raw RRR sets (immx_pool)."""

    def __init__(self, device: Device | None = None):
        self.device = device or default_device()
        h = C.c_void_p()
        check(lib.immx_pool_create(self.device.h, C.byref(h)))
        self.h = h
        self._owned = True

    @classmethod
    def borrowed(cls, handle, device):
        self = cls.__new__(cls)
        self.h, self.device, self._owned = handle, device, False
        return self

    def __del__(self):
        try:
            if self.h and self._owned:
                lib.immx_pool_destroy(self.h)
        except Exception:
            pass

    def sample(self, dg: DeviceGraph, count: int, first: int = 0, seed: int = 42, model: int = _capi.MODEL_IC):
        check(lib.immx_pool_sample(self.h, dg.h, count, first, seed, model))

    def sample_rooted(self, dg: DeviceGraph, roots, states, model: int = _capi.MODEL_IC):
        """Samples from explicit roots and raw Rng states; returns per sample the index of the
        next unused draw of its stream (draws consumed = next_draw - 1)."""
        r, s = arr(roots, np.uint32), arr(states, np.uint64)
        nd = np.zeros(max(r.size, 1), np.uint64)
        check(lib.immx_pool_sample_rooted(self.h, dg.h, ptr(r, C.c_uint32), ptr(s, C.c_uint64), r.size, model,
                                          ptr(nd, C.c_uint64)))
        return nd[: r.size]

    def upload(self, sets):
        off, mem = _sets_csr(sets)
        check(lib.immx_pool_upload(self.h, ptr(off, C.c_uint64), ptr(mem, C.c_uint32), off.size - 1))

    def info(self):
        c, m, e = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(lib.immx_pool_info(self.h, C.byref(c), C.byref(m), C.byref(e)))
        return {"count": c.value, "members": m.value, "edges": e.value}

    def __len__(self):
        return self.info()["count"]

    def read(self, lo: int = 0, hi: int | None = None):
        """-> (offsets u64[hi-lo+1], members u32[])"""
        if hi is None:
            hi = len(self)
        off = np.zeros(hi - lo + 1, np.uint64)
        # size the member buffer from an upper bound: the pool total
        mem = np.zeros(max(self.info()["members"], 1), np.uint32)
        check(lib.immx_pool_read(self.h, lo, hi, ptr(off, C.c_uint64), ptr(mem, C.c_uint32)))
        return off, mem[: int(off[-1])].copy()

    def histogram(self, n: int, lo: int = 0, hi: int | None = None) -> np.ndarray:
        if hi is None:
            hi = len(self)
        out = np.zeros(max(n, 1), np.uint64)
        check(lib.immx_pool_histogram(self.h, lo, hi, n, ptr(out, C.c_uint64)))
        return out[:n]


def _sets_csr(sets):
    off = np.zeros(len(sets) + 1, np.uint64)
    for i, s in enumerate(sets):
        if len(s) == 0:
            raise ValueError("a set must contain its root")  # module.cpp:24
        off[i + 1] = off[i] + len(s)
    mem = np.zeros(max(int(off[-1]), 1), np.uint32)
    p = 0
    for s in sets:
        mem[p:p + len(s)] = s
        p += len(s)
    return off, mem[: int(off[-1])] if off[-1] else np.zeros(0, np.uint32)


def _split(off, mem):
    off = off.astype(np.int64)
    return [mem[off[i]:off[i + 1]].tolist() for i in range(off.size - 1)]


# ------------------------------------------------------------------------ scalars
def theta_bound(n: int, k: int, epsilon: float, i: int) -> int:
    out = C.c_uint64()
    check(lib.immx_theta_bound(n, k, epsilon, i, C.byref(out)))
    return out.value


def theta_bound_real(n: int, k: int, epsilon: float, i: int) -> float:
    out = C.c_double()
    check(lib.immx_theta_bound_real(n, k, epsilon, i, C.byref(out)))
    return out.value


def skewness(sizes) -> float:
    s = arr(sizes, np.uint32)
    out = C.c_double()
    check(lib.immx_skewness(ptr(s, C.c_uint32), s.size, C.byref(out)))
    return out.value


def density(sizes, n: int) -> float:
    s = arr(sizes, np.uint32)
    out = C.c_double()
    check(lib.immx_density(ptr(s, C.c_uint32), s.size, n, C.byref(out)))
    return out.value


def choose_encoding(skewness: float, density: float) -> str:
    return _MODE_NAME[lib.immx_choose_encoding(skewness, density)]


# ------------------------------------------------------------------------ sampling
def _device_gt(g_t: Graph) -> DeviceGraph:
    return DeviceGraph(g_t, transposed=True)


def sample_rrr(g_t: Graph, root: int, seed: int):
    """module.cpp:110-116: raw Rng(seed) (not stream_for), on the device."""
    dg = _device_gt(g_t)
    if root >= dg.n:
        raise IndexError("root out of range")
    pool = Pool(dg.device)
    pool.sample_rooted(dg, [root], [seed])
    off, mem = pool.read()
    return mem.tolist()


def sample_block(g_t: Graph, count: int, first_index: int = 0, block_index: int = 1, seed: int = 42,
                 workers: int = 1):
    """sampler.cpp:85-104 -> list of member lists (visit order, root first)."""
    dg = _device_gt(g_t)
    pool = Pool(dg.device)
    pool.sample(dg, count, first_index, seed)
    off, mem = pool.read()
    return _split(off, mem)


def estimate_theta(g_t: Graph, k: int, epsilon: float, seed: int = 42, workers: int = 1):
    dg = _device_gt(g_t)
    plan = _capi.immx_plan()
    check(lib.immx_estimate_theta(dg.h, k, epsilon, seed, _capi.MODEL_IC, None, C.byref(plan)))
    return {"theta": plan.theta, "exit_iteration": plan.exit_iteration, "covered_fraction": plan.covered_fraction,
            "estimation_samples": plan.estimation_samples}


# ------------------------------------------------------------------------- huffman
class HuffmanCodebook:
    """huffman.hpp:14-31: codes per vertex; a device store is attached lazily for encode/decode."""

    def __init__(self, bits: np.ndarray, lens: np.ndarray, coded: int):
        self.bits, self.lens, self.coded_vertices = bits, lens, coded
        self._store = None

    def has_code(self, v: int) -> bool:
        return bool(self.lens[v] != 0)

    def code_length(self, v: int) -> int:
        return int(self.lens[v])

    def dump(self) -> str:
        out = []
        for v in np.nonzero(self.lens)[0]:
            ln = int(self.lens[v])
            out.append(f"{v} {ln} {format(int(self.bits[v]), 'b').zfill(ln)}\n")
        return "".join(out)

    def store(self):
        if self._store is None:
            self._store = Store(self)
        return self._store


class Store:
    """Device Huffman store (immx_store) bound to a codebook."""

    def __init__(self, cb: HuffmanCodebook, device: Device | None = None, handle=None):
        self.device = device or default_device()
        self.cb = cb
        if handle is not None:
            self.h, self._owned = handle, False
            return
        h = C.c_void_p()
        check(lib.immx_store_create(self.device.h, cb.lens.size, ptr(cb.bits, C.c_uint64), ptr(cb.lens, C.c_uint8),
                                    C.byref(h)))
        self.h, self._owned = h, True

    def __del__(self):
        try:
            if self.h and self._owned:
                lib.immx_store_destroy(self.h)
        except Exception:
            pass

    def decode_find(self, j: int, top: int):
        """huffman.cpp:129-158 on stored set j -> (found, decoded); a hybrid bitmap set is a
        bit test and decodes nothing."""
        found, nd = C.c_int(), C.c_uint64()
        bo, _, bl, _, _ = self.read(j, j + 1)
        cap = 1 if int(bl[0]) == 2 ** 64 - 1 else int(bl[0]) + 1
        dec = np.zeros(cap, np.uint32)
        check(lib.immx_store_decode_find(self.h, j, top, C.byref(found), ptr(dec, C.c_uint32), C.byref(nd)))
        return bool(found.value), dec[: nd.value].tolist()

    def encode(self, pool: "Pool", lo: int, hi: int, top=None):
        """huffman.cpp:107-127 for sets [lo, hi) of a device pool, appended to the store."""
        check(lib.immx_store_encode(self.h, pool.h, lo, hi, -1 if top is None else int(top)))

    def append(self, bits: bytes, bit_length: int, copied=()):
        """One EncodedRrr from host bytes (huffman.hpp:39-45), appended as is."""
        b = np.frombuffer(bits, np.uint8).copy() if bits else np.zeros(0, np.uint8)
        cp = arr(copied, np.uint32)
        check(lib.immx_store_append(self.h, ptr(b, C.c_uint8), b.size, int(bit_length), ptr(cp, C.c_uint32), cp.size))

    def set_hybrid(self, enable: bool = True):
        """Per-set hybrid (extension): later-encoded sets above n/32 become n-bit bitmaps."""
        check(lib.immx_store_set_hybrid(self.h, int(bool(enable))))

    def info(self):
        c, p, d = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(lib.immx_store_info(self.h, C.byref(c), C.byref(p), C.byref(d)))
        return {"count": c.value, "payload_bytes": p.value, "device_bytes": d.value}

    def codebook(self, n: int):
        """(code_bits u64[n], code_len u8[n]) of the store's codebook (len 0: uncoded, bits 0)."""
        bits, lens = np.zeros(n, np.uint64), np.zeros(n, np.uint8)
        check(lib.immx_store_codebook(self.h, ptr(bits, C.c_uint64), ptr(lens, C.c_uint8)))
        return bits, lens

    def read(self, lo: int, hi: int):
        cnt = hi - lo
        bo = np.zeros(cnt + 1, np.uint64)
        bl = np.zeros(max(cnt, 1), np.uint64)
        co = np.zeros(cnt + 1, np.uint64)
        check(lib.immx_store_read(self.h, lo, hi, ptr(bo, C.c_uint64), None, ptr(bl, C.c_uint64),
                                  ptr(co, C.c_uint64), None))
        by = np.zeros(max(int(bo[-1]), 1), np.uint8)
        cp = np.zeros(max(int(co[-1]), 1), np.uint32)
        check(lib.immx_store_read(self.h, lo, hi, None, ptr(by, C.c_uint8), None, None, ptr(cp, C.c_uint32)))
        return bo, by[: int(bo[-1])], bl[:cnt], co, cp[: int(co[-1])]


class EncodedRrr:
    """huffman.hpp:39-45"""

    def __init__(self, bits: bytes, bit_length: int, copied):
        self.bits, self.bit_length, self.copied = bits, int(bit_length), list(copied)

    def payload_bytes(self) -> int:
        return len(self.bits) + 4 * len(self.copied)

    def __repr__(self):
        return f"EncodedRrr(bit_length={self.bit_length}, copied={self.copied})"


def build_codebook(sets, n: int) -> HuffmanCodebook:
    """huffman.cpp:86-92: vertex histogram of the sets on the device, tree on the host."""
    if len(sets) == 0:
        raise RuntimeError("cannot build a codebook from an empty block")
    pool = Pool()
    pool.upload(sets)
    freq = pool.histogram(n)
    return codebook_from_counts(freq)


def codebook_from_counts(freq) -> HuffmanCodebook:
    f = arr(freq, np.uint64)
    bits = np.zeros(max(f.size, 1), np.uint64)
    lens = np.zeros(max(f.size, 1), np.uint8)
    coded = C.c_uint64()
    check(lib.immx_codebook_build(ptr(f, C.c_uint64), f.size, ptr(bits, C.c_uint64), ptr(lens, C.c_uint8),
                                  C.byref(coded)))
    return HuffmanCodebook(bits[: f.size], lens[: f.size], coded.value)


def encode_rrr(codebook: HuffmanCodebook, members, top=None) -> EncodedRrr:
    """huffman.cpp:107-127 on the device."""
    st = codebook.store()
    pool = Pool(st.device)
    pool.upload([list(members)]) if len(members) else None
    if len(members) == 0:
        return EncodedRrr(b"", 0, [])
    j = st.info()["count"]
    check(lib.immx_store_encode(st.h, pool.h, 0, 1, -1 if top is None else int(top)))
    bo, by, bl, co, cp = st.read(j, j + 1)
    return EncodedRrr(bytes(by), int(bl[0]), cp.tolist())


def decode_find(codebook: HuffmanCodebook, encoded: EncodedRrr, top: int):
    """huffman.cpp:129-158 on the device -> (found, decoded)."""
    st = codebook.store()
    b = np.frombuffer(encoded.bits, np.uint8).copy() if encoded.bits else np.zeros(0, np.uint8)
    cp = arr(encoded.copied, np.uint32)
    check(lib.immx_store_append(st.h, ptr(b, C.c_uint8), b.size, encoded.bit_length, ptr(cp, C.c_uint32), cp.size))
    j = st.info()["count"] - 1
    found = C.c_int()
    dec = np.zeros(encoded.bit_length + 1, np.uint32)
    nd = C.c_uint64()
    check(lib.immx_store_decode_find(st.h, j, top, C.byref(found), ptr(dec, C.c_uint32), C.byref(nd)))
    return bool(found.value), dec[: nd.value].tolist()


# -------------------------------------------------------------------------- bitmap
class BitmapCollection:
    """bitmap.hpp:31-51 on the device (immx_bitmap)."""

    def __init__(self, n_rows: int, device: Device | None = None):
        self.device = device or default_device()
        h = C.c_void_p()
        check(lib.immx_bitmap_create(self.device.h, n_rows, C.byref(h)))
        self.h = h
        self.n_rows = n_rows
        self._blocks = []

    def __del__(self):
        try:
            if self.h:
                lib.immx_bitmap_destroy(self.h)
        except Exception:
            pass

    def _info(self):
        c, w, b, nb = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint32()
        check(lib.immx_bitmap_info(self.h, C.byref(c), C.byref(w), C.byref(b), C.byref(nb)))
        return c.value, w.value, b.value, nb.value

    @property
    def n_cols(self) -> int:
        return self._info()[0]

    def byte_size(self) -> int:
        return self._info()[2]

    def popcounts(self) -> np.ndarray:
        out = np.zeros(max(self.n_rows, 1), np.uint64)
        check(lib.immx_bitmap_popcount(self.h, ptr(out, C.c_uint64)))
        return out[: self.n_rows]

    def popcount_row(self, v: int) -> int:
        if v >= self.n_rows:
            raise IndexError("row out of range")
        return int(bin(0).count("1") + sum(bin(int(w)).count("1") for w in self.snapshot_row(v)))

    def snapshot_row(self, v: int):
        w = np.zeros(max(self._info()[1], 1), np.uint32)
        check(lib.immx_bitmap_row(self.h, v, ptr(w, C.c_uint32)))
        return w[: self._info()[1]].tolist()

    def subtract_row(self, v: int, top: int) -> int:
        """bitmap.cpp:66-69: the live-row convenience form (snapshot of top taken now)."""
        snap = arr(self.snapshot_row(top), np.uint32)
        pc = C.c_uint64()
        check(lib.immx_bitmap_subtract_row(self.h, v, ptr(snap, C.c_uint32), C.byref(pc)))
        return pc.value

    def subtract_snapshot(self, v: int, snapshot) -> int:
        snap = arr(snapshot, np.uint32)
        pc = C.c_uint64()
        check(lib.immx_bitmap_subtract_row(self.h, v, ptr(snap, C.c_uint32), C.byref(pc)))
        return pc.value

    def row_bits(self, v: int):
        words = self.snapshot_row(v)
        bits, base = [], 0
        for cols in self._blocks:
            wpr = (cols + 31) // 32
            for c in range(cols):
                bits.append((words[base + c // 32] >> (c % 32)) & 1)
            base += wpr
        return bits


def encode_bitmap(sets, n: int) -> BitmapCollection:
    pool = Pool()
    pool.upload(sets)
    bm = BitmapCollection(n, pool.device)
    check(lib.immx_bitmap_encode_block(bm.h, pool.h, 0, len(sets)))
    bm._blocks.append(len(sets))
    return bm


# ----------------------------------------------------------------------- selection
def _sel_arrays(k):
    return np.zeros(k, np.uint32), np.zeros(k, np.uint64), np.zeros(k, np.float64), C.c_uint32()


def _sel_dict(seeds, marg, cov, padded):
    return {"seeds": seeds.tolist(), "marginal": marg.tolist(), "coverage": cov.tolist(), "padded": padded.value}


def _check_merged(merged: bool, workers: int) -> None:
    """select.cpp:71-74: with merged_argmax and more than one worker the reference picks from
    the per-chunk winners only (a heuristic, not the exact argmax).  That mode is out of scope
    here, so it is refused rather than silently answered exactly; with one
    worker the reference itself falls back to the exact argmax, and so does this."""
    if merged and workers > 1:
        raise ValueError("merged_argmax with workers > 1 (the reference's per-chunk heuristic pick) is not "
                         "supported by the B200 path, which selects with the exact argmax")


def select_raw(sets, n: int, k: int, workers: int = 1, merged_argmax: bool = False):
    """select.cpp:89-148 with the exact argmax (ties -> lowest id).  merged_argmax=True with
    workers > 1 raises ValueError (see _check_merged)."""
    _check_merged(merged_argmax, workers)
    if len(sets) == 0:
        raise ValueError("selection requires at least one set")
    pool = Pool()
    pool.upload(sets)
    s, m, c, p = _sel_arrays(k)
    check(lib.immx_select_raw(pool.h, n, k, ptr(s, C.c_uint32), ptr(m, C.c_uint64), ptr(c, C.c_double), C.byref(p)))
    return _sel_dict(s, m, c, p)


def select_huffman(codebook: HuffmanCodebook, store: Store, hist, k: int):
    h = arr(hist, np.uint64)
    s, m, c, p = _sel_arrays(k)
    md = np.zeros(k, np.uint64)
    check(lib.immx_select_huffman(store.h, ptr(h, C.c_uint64), k, ptr(s, C.c_uint32), ptr(m, C.c_uint64),
                                  ptr(c, C.c_double), C.byref(p), ptr(md, C.c_uint64)))
    d = _sel_dict(s, m, c, p)
    d["max_decoded"] = md.tolist()
    return d


def select_bitmap(bm: BitmapCollection, k: int, hist=None):
    h = None if hist is None else arr(hist, np.uint64)
    s, m, c, p = _sel_arrays(k)
    check(lib.immx_select_bitmap(bm.h, ptr(h, C.c_uint64), k, ptr(s, C.c_uint32), ptr(m, C.c_uint64),
                                 ptr(c, C.c_double), C.byref(p)))
    return _sel_dict(s, m, c, p)


def table_argmax(counts) -> int:
    c = arr(counts, np.uint64)
    out = C.c_uint32()
    check(lib.immx_table_argmax(default_device().h, ptr(c, C.c_uint64), c.size, C.byref(out)))
    return out.value


def merged_argmax(locals):
    """select.cpp:22-43 -- the reduced-candidate heuristic (k*p values).  A host-side utility
    kept for API parity; it is not on the exact hot path."""
    if len(locals) == 0:
        raise ValueError("merged_argmax needs at least one table")
    winners = sorted({table_argmax(t) for t in locals})
    best, best_count = winners[0], 0
    for w in winners:
        total = sum(int(t[w]) for t in locals)
        if total > best_count or (total == best_count and w < best):
            best, best_count = w, total
    return best


# ----------------------------------------------------------------------------- run
def run_device(dg: DeviceGraph, k: int, *, epsilon=0.5, blocks=8, mode="auto", seed=42, workers=1,
               model: int = _capi.MODEL_IC, reuse_pool: bool = True, keep: bool = False):
    """pipeline.cpp:47-178 on a graph already resident in HBM.  Returns the raw result dict."""
    cfg = _capi.immx_run_config(k, epsilon, blocks, -1 if mode == "auto" else _MODE_ID[mode], seed, workers, model,
                                int(reuse_pool))
    h = C.c_void_p()
    check(lib.immx_run(dg.h, C.byref(cfg), C.byref(h)))
    try:
        st = _capi.immx_run_stats()
        st.struct_size = C.sizeof(st)
        check(lib.immx_result_stats(h, C.byref(st)))
        if st.version != _capi.RUN_STATS_VERSION:
            raise RuntimeError(f"immx_run_stats version {st.version}, expected {_capi.RUN_STATS_VERSION}")
        seeds, marg, cov = np.zeros(k, np.uint32), np.zeros(k, np.uint64), np.zeros(k, np.float64)
        check(lib.immx_result_seeds(h, ptr(seeds, C.c_uint32), ptr(marg, C.c_uint64), ptr(cov, C.c_double)))
        b = int(st.blocks)
        bs, br, be = np.zeros(b, np.uint64), np.zeros(b, np.uint64), np.zeros(b, np.uint64)
        check(lib.immx_result_blocks(h, ptr(bs, C.c_uint64), ptr(br, C.c_uint64), ptr(be, C.c_uint64)))
        out = {
            "seeds": seeds.tolist(), "marginal": marg.tolist(), "coverage": cov.tolist(), "padded": st.padded,
            "theta": st.theta, "estimation_samples": st.estimation_samples, "exit_iteration": st.exit_iteration,
            "blocks": b, "raw_bytes": st.raw_bytes, "encoded_bytes": st.encoded_bytes, "peak_bytes": st.peak_bytes,
            "coded_vertices": st.coded_vertices, "device_store_bytes": st.device_store_bytes,
            "samples_drawn": st.samples_drawn, "edges_scanned": st.edges_scanned, "pool_members": st.members,
            "dense_sets": st.dense_sets, "covered_fraction": st.covered_fraction, "skewness": st.skewness,
            "density": st.density, "compression_ratio": st.compression_ratio,
            "uncoded_vertex_fraction": st.uncoded_vertex_fraction,
            "phase_seconds": {"estimate": st.t_estimate, "sample_encode": st.t_sample_encode, "select": st.t_select,
                              "total": st.t_total},
            "host_seconds": {"codebook": st.t_codebook, "decode_table": st.t_decode_table},
            "characterized_mode": _MODE_NAME[st.characterized_mode], "mode": _MODE_NAME[st.mode],
            "mode_override": bool(st.mode_overridden),
            "device_peak_bytes": st.device_peak_bytes, "device_resident_bytes": st.device_resident_bytes,
            "device_graph_bytes": st.device_graph_bytes,
            "block_sets": bs.tolist(), "block_raw": br.tolist(), "block_enc": be.tolist(),
        }
        if keep:
            out["_store"] = (Store(None, dg.device, handle=lib.immx_result_store(h))
                             if out["mode"] in ("huffman", "hybrid") else None)
        return out
    finally:
        if not keep:
            lib.immx_result_destroy(h)


def run(graph: Graph, k: int, *, epsilon=0.5, blocks=8, mode="auto", seed=42, workers=1, merged_argmax=False,
        reuse_pool=True, diffusion="ic", lt_seed=0, lt_weights=None):
    """The IMM driver (pipeline.cpp:47-178) -> {seeds, marginal, coverage, padded, seed_ids, stats}.
    The graph (forward) is uploaded and transposed on the device.  diffusion="lt" (extension,
    no reference counterpart) samples reverse LT walks with `lt_weights` (per Gt edge) or the
    generator's weights for `lt_seed`."""
    n = graph.n
    if k < 1 or k >= n:
        raise ValueError("k must satisfy 1 <= k < n")
    if not epsilon > 0:
        raise ValueError("epsilon must be > 0")
    if blocks < 2:
        raise ValueError("block count must be >= 2")
    if mode != "auto" and mode not in _MODE_ID:
        raise ValueError(f"unknown mode '{mode}'")
    if diffusion not in ("ic", "lt"):
        raise ValueError(f"unknown diffusion model '{diffusion}'")
    _check_merged(merged_argmax, workers)
    dg = DeviceGraph(graph, transposed=False)
    model = _capi.MODEL_IC
    if diffusion == "lt":
        model = _capi.MODEL_LT
        if lt_weights is not None:
            dg.set_lt_weights(lt_weights)
        else:
            dg.set_lt_random(lt_seed)
    r = run_device(dg, k, epsilon=epsilon, blocks=blocks, mode=mode, seed=seed, workers=workers,
                   reuse_pool=reuse_pool, model=model)
    ids = graph.original_ids
    theta = r["theta"]
    stats = {
        "n": n, "m": graph.m, "theta": theta, "skewness": r["skewness"], "density": r["density"],
        "mode": r["mode"], "mode_override": r["mode_override"], "phase_seconds": r["phase_seconds"],
        "raw_bytes": r["raw_bytes"], "encoded_bytes": r["encoded_bytes"],
        "compression_ratio": r["compression_ratio"], "peak_bytes": r["peak_bytes"],
        "padded_seeds": r["padded"], "uncoded_vertex_fraction": r["uncoded_vertex_fraction"],
        "blocks": [{"sets": s, "raw_bytes": a, "encoded_bytes": e}
                   for s, a, e in zip(r["block_sets"], r["block_raw"], r["block_enc"])],
        "seeds": [{"id": int(ids[s]), "marginal": mg / theta, "cumulative": cv}
                  for s, mg, cv in zip(r["seeds"], r["marginal"], r["coverage"])],
        "plan": {"k": k, "epsilon": epsilon, "blocks": r["blocks"], "rng_seed": seed, "workers": workers,
                 "exit_iteration": r["exit_iteration"], "estimation_samples": r["estimation_samples"],
                 "covered_fraction": r["covered_fraction"]},
        "original_ids": ids.tolist(),
        "rss_bytes": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss * 1024,
        "device": {"samples_drawn": r["samples_drawn"], "edges_scanned": r["edges_scanned"],
                   "device_store_bytes": r["device_store_bytes"], "coded_vertices": r["coded_vertices"],
                   "dense_sets": r["dense_sets"]},
    }
    return {"seeds": r["seeds"], "marginal": r["marginal"], "coverage": r["coverage"], "padded": r["padded"],
            "seed_ids": [int(ids[s]) for s in r["seeds"]], "stats": stats}


# ----------------------------------------------------------------------------- stats output
_STATS_KEYS = ("n", "m", "theta", "skewness", "density", "mode", "mode_override", "phase_seconds", "raw_bytes",
               "encoded_bytes", "compression_ratio", "peak_bytes", "padded_seeds", "uncoded_vertex_fraction",
               "blocks", "seeds", "plan", "original_ids", "rss_bytes")


def stats_to_json(stats: dict) -> str:
    """stats_json.cpp:21-72: the run stats (the dict ``run`` returns) in the reference's schema
    and key order, 2-space indented.  The device-only counters (``stats["device"]``) are not
    part of that schema and are left out."""
    import json

    out = {key: stats[key] for key in _STATS_KEYS}
    out["rss_bytes"] = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss * 1024  # informational
    return json.dumps(out, indent=2)


def write_stats(stats: dict, path: str) -> None:
    """stats_json.cpp:74-79"""
    try:
        with open(path, "w") as f:
            f.write(stats_to_json(stats) + "\n")
    except OSError as e:
        raise RuntimeError(f"cannot write stats to '{path}'") from e


def write_seeds(stats: dict, path: str) -> None:
    """stats_json.cpp:81-86: one original vertex id per line"""
    try:
        with open(path, "w") as f:
            for s in stats["seeds"]:
                f.write(f"{s['id']}\n")
    except OSError as e:
        raise RuntimeError(f"cannot write seeds to '{path}'") from e
