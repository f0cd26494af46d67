"""ctypes front-end for the parity checkers in oracle/.

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs.  The product package never imports this.

* ``Oracle``  -- the C restatement (oracle/immx_oracle.c -> oracle/liboracle.so).
* ``RefLib``  -- the unmodified reference compiled from its sources
  (oracle/_ref/libimmx_ref.so, recipe oracle/Makefile), when present.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libimmx_ref.so")

u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")

MODES = {"huffman": 0, "bitmap": 1, "raw": 2, "hybrid": 3}  # 3: builder extension (per-set hybrid)
MODE_NAMES = {v: k for k, v in MODES.items()}


@dataclass
class CSR:
    """A graph as plain CSR arrays (forward or transposed, as the caller says)."""

    n: int
    off: np.ndarray  # u64[n+1]
    tgt: np.ndarray  # u32[m]
    prob: np.ndarray  # f64[m]

    @property
    def m(self) -> int:
        return int(self.tgt.shape[0])


def _sig(lib, name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args
    return f


class Oracle:
    def __init__(self, path: str = LIB_PATH):
        if not os.path.exists(path):
            raise RuntimeError(f"oracle library missing: {path} (run make -C oracle)")
        L = self.L = C.CDLL(path)
        V, P = C.c_void_p, C.c_void_p
        _sig(L, "oc_mix64", C.c_uint64, [C.c_uint64])
        _sig(L, "oc_stream_state", C.c_uint64, [C.c_uint64, C.c_uint64])
        _sig(L, "oc_transpose", None, [C.c_uint64, C.c_uint64, u64p, u32p, f64p, u64p, u32p, f64p])
        _sig(L, "oc_assign_weights", None, [C.c_uint64, C.c_uint64, u32p, f64p, C.c_int, C.c_double])
        _sig(L, "oc_sample_block", P, [C.c_uint64, u64p, u32p, f64p, C.c_uint64, C.c_uint64, C.c_uint64])
        _sig(L, "oc_sample_block_lt", P, [C.c_uint64, u64p, u32p, f32p, C.c_uint64, C.c_uint64, C.c_uint64])
        _sig(L, "oc_block_count", C.c_uint64, [P])
        _sig(L, "oc_block_total", C.c_uint64, [P])
        _sig(L, "oc_block_edges", C.c_uint64, [P])
        _sig(L, "oc_block_copy", None, [P, u64p, u32p])
        _sig(L, "oc_block_free", None, [P])
        _sig(L, "oc_sample_rrr_seed", C.c_int64,
             [C.c_uint64, u64p, u32p, f64p, C.c_uint32, C.c_uint64, u32p, C.c_uint64])
        _sig(L, "oc_theta_base", C.c_double, [C.c_uint64, C.c_uint64, C.c_double])
        _sig(L, "oc_theta_bound_real", C.c_double, [C.c_uint64, C.c_uint64, C.c_double, C.c_uint32])
        _sig(L, "oc_theta_bound", C.c_uint64, [C.c_uint64, C.c_uint64, C.c_double, C.c_uint32])
        _sig(L, "oc_table_argmax", C.c_uint32, [u64p, C.c_uint64])
        _sig(L, "oc_select_raw", C.c_uint32, [u64p, u32p, C.c_uint64, C.c_uint64, C.c_uint32, u32p, u64p, f64p])
        _sig(L, "oc_estimate_theta", None,
             [C.c_uint64, u64p, u32p, f64p, C.c_uint32, C.c_double, C.c_uint64, u64p, C.POINTER(C.c_double)])
        _sig(L, "oc_skewness", C.c_double, [u32p, C.c_uint64])
        _sig(L, "oc_density", C.c_double, [u32p, C.c_uint64, C.c_uint64])
        _sig(L, "oc_choose_encoding", C.c_int, [C.c_double, C.c_double])
        _sig(L, "oc_build_codebook", P, [u64p, C.c_uint64])
        _sig(L, "oc_codebook_error", C.c_int, [P])
        _sig(L, "oc_codebook_coded", C.c_uint64, [P])
        _sig(L, "oc_codebook_codes", None, [P, u64p, u8p])
        _sig(L, "oc_codebook_free", None, [P])
        _sig(L, "oc_encode_rrr", C.c_uint64, [P, u32p, C.c_uint64, C.c_int64, u8p, u32p, C.POINTER(C.c_uint64)])
        _sig(L, "oc_decode_find", C.c_int,
             [P, u8p, C.c_uint64, C.c_uint64, u32p, C.c_uint64, C.c_uint32, u32p, C.POINTER(C.c_uint64)])
        _sig(L, "oc_store_build", P, [P, u64p, u32p, C.c_uint64, C.c_int64])
        _sig(L, "oc_store_sizes", None, [P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)])
        _sig(L, "oc_store_copy", None, [P, u64p, u64p, u8p, u64p, u32p])
        _sig(L, "oc_store_free", None, [P])
        _sig(L, "oc_select_huffman", C.c_uint32, [P, P, u64p, C.c_uint64, C.c_uint32, u32p, u64p, f64p, u64p])
        _sig(L, "oc_bitmap_encode", None, [u64p, u32p, C.c_uint64, C.c_uint64, C.c_uint64, u32p])
        _sig(L, "oc_select_bitmap", C.c_uint32,
             [u32p, u64p, u64p, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint32, u32p, u64p, f64p])
        _sig(L, "oc_run", P, [C.c_uint64, C.c_uint64, u64p, u32p, f64p, C.c_uint32, C.c_double,
                              C.c_uint32, C.c_int, C.c_uint64, C.c_int])
        _sig(L, "oc_run_lt", P, [C.c_uint64, C.c_uint64, u64p, u32p, f64p, f32p, C.c_uint32, C.c_double,
                                 C.c_uint32, C.c_int, C.c_uint64, C.c_int])
        _sig(L, "oc_estimate_theta_lt", None,
             [C.c_uint64, u64p, u32p, f32p, C.c_uint32, C.c_double, C.c_uint64, u64p, C.POINTER(C.c_double)])
        _sig(L, "oc_run_scalars", None, [P, u64p, f64p, i32p])
        _sig(L, "oc_run_seeds", None, [P, u32p, u64p, f64p])
        _sig(L, "oc_run_blocks", None, [P, u64p, u64p, u64p, u32p])
        _sig(L, "oc_run_pool", None, [P, u64p, u32p])
        _sig(L, "oc_run_store", None, [P, u64p, u64p, u8p, u64p, u32p])
        _sig(L, "oc_run_codebook", P, [P])
        _sig(L, "oc_run_free", None, [P])
        _sig(L, "og_rmat", P, [C.c_uint32, C.c_uint32, C.c_double, C.c_double, C.c_double, C.c_uint64, C.c_int])
        _sig(L, "og_er", P, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int])
        _sig(L, "og_csr_n", C.c_uint64, [P])
        _sig(L, "og_csr_m", C.c_uint64, [P])
        _sig(L, "og_csr_offsets", C.POINTER(C.c_uint64), [P])
        _sig(L, "og_csr_targets", C.POINTER(C.c_uint32), [P])
        _sig(L, "og_csr_free", None, [P])
        _sig(L, "og_weights_f32", None, [P, C.c_int, C.c_int, C.c_double, f64p])
        _sig(L, "og_lt_weights", None, [P, C.c_uint64, f32p])

    # ---------------------------------------------------- config graphs (gen_graph.c)
    def generate(self, gen, weights=("wc", 0.0), reverse: bool = True, lt_seed=None):
        """A BASELINE-config graph from oracle/gen_graph.c: gen = ("rmat", scale, ef, seed) or
        ("er", n, m, seed); weights = (model, p) as float32-rounded doubles.  reverse=True gives
        G^T.  With lt_seed (reverse only) also returns the LT weights (f32 per G^T edge)."""
        L = self.L
        h = (L.og_rmat(gen[1], gen[2], 0.57, 0.19, 0.19, gen[3], int(reverse)) if gen[0] == "rmat"
             else L.og_er(gen[1], gen[2], gen[3], int(reverse)))
        if not h:
            raise ValueError("generator arguments out of range")
        try:
            n, m = L.og_csr_n(h), L.og_csr_m(h)
            off = np.ctypeslib.as_array(L.og_csr_offsets(h), shape=(n + 1,)).copy()
            tgt = np.ctypeslib.as_array(L.og_csr_targets(h), shape=(max(m, 1),))[:m].copy()
            prob = np.zeros(max(m, 1), np.float64)
            L.og_weights_f32(h, int(reverse), 0 if weights[0] == "wc" else 1, float(weights[1]), prob)
            g = CSR(n, off, tgt, prob[:m])
            if lt_seed is None:
                return g
            w = np.zeros(max(m, 1), np.float32)
            L.og_lt_weights(h, lt_seed, w)
            return g, w[:m]
        finally:
            L.og_csr_free(h)

    # ---------------------------------------------------------------- RNG
    def mix64(self, z: int) -> int:
        return self.L.oc_mix64(z)

    def stream_state(self, seed: int, index: int) -> int:
        return self.L.oc_stream_state(seed, index)

    # -------------------------------------------------------------- graph
    def transpose(self, g: CSR) -> CSR:
        off = np.zeros(g.n + 1, np.uint64)
        tgt = np.zeros(max(g.m, 1), np.uint32)
        prob = np.zeros(max(g.m, 1), np.float64)
        self.L.oc_transpose(g.n, g.m, g.off, g.tgt, g.prob, off, tgt, prob)
        return CSR(g.n, off, tgt[: g.m].copy(), prob[: g.m].copy())

    def assign_weights(self, g: CSR, model: str = "wc", p: float = 0.1) -> CSR:
        prob = np.zeros(max(g.m, 1), np.float64)
        self.L.oc_assign_weights(g.n, g.m, g.tgt if g.m else np.zeros(1, np.uint32), prob,
                                 0 if model == "wc" else 1, p)
        return CSR(g.n, g.off, g.tgt, prob[: g.m].copy())

    # ------------------------------------------------------------ sampling
    def _take_block(self, h):
        cnt = self.L.oc_block_count(h)
        tot = self.L.oc_block_total(h)
        edges = self.L.oc_block_edges(h)
        offs = np.zeros(cnt + 1, np.uint64)
        mem = np.zeros(max(tot, 1), np.uint32)
        self.L.oc_block_copy(h, offs, mem)
        self.L.oc_block_free(h)
        return offs, mem[:tot].copy(), edges

    def sample_block(self, gt: CSR, count: int, first: int = 0, seed: int = 42):
        """-> (offsets u64[count+1], members u32[], edges_scanned)."""
        h = self.L.oc_sample_block(gt.n, gt.off, _nz32(gt.tgt), _nz64(gt.prob), count, first, seed)
        return self._take_block(h)

    def sample_block_lt(self, gt: CSR, weights: np.ndarray, count: int, first: int = 0, seed: int = 42):
        w = np.ascontiguousarray(weights, np.float32)
        h = self.L.oc_sample_block_lt(gt.n, gt.off, _nz32(gt.tgt), w if w.size else np.zeros(1, np.float32),
                                      count, first, seed)
        return self._take_block(h)

    def sample_rrr(self, gt: CSR, root: int, seed: int):
        out = np.zeros(gt.n + 1, np.uint32)
        r = self.L.oc_sample_rrr_seed(gt.n, gt.off, _nz32(gt.tgt), _nz64(gt.prob), root, seed, out, gt.n + 1)
        return out[:r].tolist()

    # --------------------------------------------------------------- theta
    def theta_bound(self, n, k, eps, i):
        return self.L.oc_theta_bound(n, k, eps, i)

    def theta_bound_real(self, n, k, eps, i):
        return self.L.oc_theta_bound_real(n, k, eps, i)

    def theta_base(self, n, k, eps):
        return self.L.oc_theta_base(n, k, eps)

    def estimate_theta(self, gt: CSR, k: int, eps: float, seed: int = 42):
        out = np.zeros(3, np.uint64)
        F = C.c_double()
        self.L.oc_estimate_theta(gt.n, gt.off, _nz32(gt.tgt), _nz64(gt.prob), k, eps, seed, out, C.byref(F))
        return {"theta": int(out[0]), "exit_iteration": int(out[1]),
                "estimation_samples": int(out[2]), "covered_fraction": F.value}

    # ----------------------------------------------------------- selection
    def table_argmax(self, counts) -> int:
        c = np.ascontiguousarray(counts, np.uint64)
        return self.L.oc_table_argmax(c if c.size else np.zeros(1, np.uint64), c.size)

    def select_raw(self, set_off, members, n: int, k: int):
        set_off = np.ascontiguousarray(set_off, np.uint64)
        members = np.ascontiguousarray(members, np.uint32)
        theta = set_off.size - 1
        seeds = np.zeros(k, np.uint32)
        marg = np.zeros(k, np.uint64)
        cov = np.zeros(k, np.float64)
        padded = self.L.oc_select_raw(set_off, _nz32(members), theta, n, k, seeds, marg, cov)
        return {"seeds": seeds.tolist(), "marginal": marg.tolist(), "coverage": cov.tolist(), "padded": padded}

    # ------------------------------------------------------- characterize
    def skewness(self, sizes):
        s = np.ascontiguousarray(sizes, np.uint32)
        return self.L.oc_skewness(s, s.size)

    def density(self, sizes, n):
        s = np.ascontiguousarray(sizes, np.uint32)
        return self.L.oc_density(s, s.size, n)

    def choose_encoding(self, s, d):
        return MODE_NAMES[self.L.oc_choose_encoding(s, d)]

    # -------------------------------------------------------------- huffman
    def codebook(self, freq) -> "OracleCodebook":
        f = np.ascontiguousarray(freq, np.uint64)
        return OracleCodebook(self, self.L.oc_build_codebook(f, f.size), f.size)

    def codebook_from_sets(self, sets, n) -> "OracleCodebook":
        f = np.zeros(n, np.uint64)
        for s in sets:
            for v in s:
                f[v] += 1
        return self.codebook(f)

    # --------------------------------------------------------------- bitmap
    def select_bitmap_sets(self, set_off, members, n: int, k: int, blocks: int = 1):
        set_off = np.ascontiguousarray(set_off, np.uint64)
        members = np.ascontiguousarray(members, np.uint32)
        theta = set_off.size - 1
        per = (theta + blocks - 1) // blocks
        words, base, wpr = [], [], []
        tot = 0
        lo = 0
        while lo < theta:
            hi = min(theta, lo + per)
            w = (hi - lo + 31) // 32
            buf = np.zeros(max(n * w, 1), np.uint32)
            self.L.oc_bitmap_encode(set_off, _nz32(members), lo, hi, n, buf)
            words.append(buf[: n * w])
            base.append(tot)
            wpr.append(w)
            tot += n * w
            lo = hi
        allw = np.ascontiguousarray(np.concatenate(words) if words else np.zeros(1, np.uint32))
        seeds = np.zeros(k, np.uint32)
        marg = np.zeros(k, np.uint64)
        cov = np.zeros(k, np.float64)
        padded = self.L.oc_select_bitmap(_nz32(allw), np.array(base, np.uint64), np.array(wpr, np.uint64),
                                         len(base), n, theta, k, seeds, marg, cov)
        return {"seeds": seeds.tolist(), "marginal": marg.tolist(), "coverage": cov.tolist(), "padded": padded}

    def bitmap_block(self, set_off, members, lo: int, hi: int, n: int) -> np.ndarray:
        w = (hi - lo + 31) // 32
        buf = np.zeros(max(n * w, 1), np.uint32)
        self.L.oc_bitmap_encode(np.ascontiguousarray(set_off, np.uint64),
                                _nz32(np.ascontiguousarray(members, np.uint32)), lo, hi, n, buf)
        return buf[: n * w].reshape(n, w) if n * w else buf[:0].reshape(n, 0)

    # ------------------------------------------------------------- pipeline
    def run(self, g: CSR, k: int, epsilon: float = 0.5, blocks: int = 8, mode: str = "auto",
            seed: int = 42, workers: int = 1, want_store: bool = False, want_pool: bool = False, lt_weights=None):
        """pipeline.cpp:47-178 on the FORWARD graph g."""
        m = -1 if mode == "auto" else MODES[mode]
        if lt_weights is not None:  # LT extension: weights per Gt edge (oc_transpose order)
            w = np.ascontiguousarray(lt_weights, np.float32)
            h = self.L.oc_run_lt(g.n, g.m, g.off, _nz32(g.tgt), _nz64(g.prob), w if w.size else np.zeros(1, np.float32),
                                 k, epsilon, blocks, m, seed, workers)
        else:
            h = self.L.oc_run(g.n, g.m, g.off, _nz32(g.tgt), _nz64(g.prob), k, epsilon, blocks, m, seed, workers)
        u = np.zeros(14, np.uint64)
        d = np.zeros(5, np.float64)
        i = np.zeros(3, np.int32)
        self.L.oc_run_scalars(h, u, d, i)
        seeds = np.zeros(k, np.uint32)
        marg = np.zeros(k, np.uint64)
        cov = np.zeros(k, np.float64)
        self.L.oc_run_seeds(h, seeds, marg, cov)
        b = int(u[3])
        bs, br, be, bt = (np.zeros(b, np.uint64), np.zeros(b, np.uint64), np.zeros(b, np.uint64),
                          np.zeros(b, np.uint32))
        self.L.oc_run_blocks(h, bs, br, be, bt)
        out = {
            "seeds": seeds.tolist(), "marginal": marg.tolist(), "coverage": cov.tolist(), "padded": int(u[7]),
            "theta": int(u[0]), "estimation_samples": int(u[1]), "exit_iteration": int(u[2]), "blocks": b,
            "raw_bytes": int(u[4]), "encoded_bytes": int(u[5]), "peak_bytes": int(u[6]),
            "coded_vertices": int(u[9]), "dense_sets": int(u[13]),
            "covered_fraction": float(d[0]), "skewness": float(d[1]), "density": float(d[2]),
            "compression_ratio": float(d[3]), "uncoded_vertex_fraction": float(d[4]),
            "characterized_mode": MODE_NAMES[int(i[0])], "mode": MODE_NAMES[int(i[1])],
            "mode_override": bool(i[2]),
            "block_sets": bs.tolist(), "block_raw": br.tolist(), "block_enc": be.tolist(), "tops": bt.tolist(),
        }
        if want_pool:
            so = np.zeros(out["theta"] + 1, np.uint64)
            mem = np.zeros(max(int(u[12]), 1), np.uint32)
            self.L.oc_run_pool(h, so, mem)
            out["pool"] = (so, mem[: int(u[12])])
        if want_store and out["mode"] in ("huffman", "hybrid"):
            t = out["theta"]
            eo, bl, cp = np.zeros(t + 1, np.uint64), np.zeros(t, np.uint64), np.zeros(t + 1, np.uint64)
            by = np.zeros(max(int(u[10]), 1), np.uint8)
            co = np.zeros(max(int(u[11]), 1), np.uint32)
            self.L.oc_run_store(h, eo, bl, by, cp, co)
            out["store"] = {"enc_off": eo, "bit_length": bl, "bytes": by[: int(u[10])], "cp_off": cp,
                            "copied": co[: int(u[11])]}
            n = g.n
            bits = np.zeros(n, np.uint64)
            lens = np.zeros(n, np.uint8)
            self.L.oc_codebook_codes(self.L.oc_run_codebook(h), bits, lens)
            out["codes"] = (bits, lens)
        self.L.oc_run_free(h)
        return out


class OracleCodebook:
    def __init__(self, orc: Oracle, h, n: int):
        self.o, self.h, self.n = orc, h, n
        self.error = orc.L.oc_codebook_error(h)
        self.coded_vertices = orc.L.oc_codebook_coded(h)
        self.bits = np.zeros(n, np.uint64)
        self.lens = np.zeros(n, np.uint8)
        if n:
            orc.L.oc_codebook_codes(h, self.bits, self.lens)

    def __del__(self):
        try:
            self.o.L.oc_codebook_free(self.h)
        except Exception:
            pass

    def code(self, v):
        ln = int(self.lens[v])
        return format(int(self.bits[v]), "b").zfill(ln) if ln else ""

    def encode(self, members, top=None):
        mem = np.ascontiguousarray(members, np.uint32)
        nbits = int(sum(int(self.lens[v]) for v in members))
        buf = np.zeros((nbits + 7) // 8 + 1, np.uint8)
        cp = np.zeros(max(len(members), 1), np.uint32)
        nc = C.c_uint64()
        bl = self.o.L.oc_encode_rrr(self.h, _nz32(mem), mem.size, -1 if top is None else int(top), buf, cp, C.byref(nc))
        return bytes(buf[: (bl + 7) // 8]), int(bl), cp[: nc.value].tolist()

    def decode_find(self, data: bytes, bit_length: int, copied, top: int):
        b = np.frombuffer(data, np.uint8).copy() if data else np.zeros(1, np.uint8)
        cp = np.ascontiguousarray(copied, np.uint32)
        out = np.zeros(bit_length + 1, np.uint32)
        nd = C.c_uint64(0)
        r = self.o.L.oc_decode_find(self.h, b, len(data), bit_length, _nz32(cp), cp.size, top, out, C.byref(nd))
        if r < 0:
            raise RuntimeError(f"corrupt payload ({r})")
        return bool(r), out[: nd.value].tolist()

    def store(self, set_off, members, top=None):
        so = np.ascontiguousarray(set_off, np.uint64)
        mem = np.ascontiguousarray(members, np.uint32)
        return OracleStore(self, self.o.L.oc_store_build(self.h, so, _nz32(mem), so.size - 1,
                                                         -1 if top is None else int(top)), so.size - 1)


class OracleStore:
    def __init__(self, cb: OracleCodebook, h, theta):
        self.cb, self.h, self.theta = cb, h, theta
        L = cb.o.L
        nb, nc = C.c_uint64(), C.c_uint64()
        L.oc_store_sizes(h, C.byref(nb), C.byref(nc))
        self.enc_off = np.zeros(theta + 1, np.uint64)
        self.bit_length = np.zeros(max(theta, 1), np.uint64)
        by = np.zeros(max(nb.value, 1), np.uint8)
        self.cp_off = np.zeros(theta + 1, np.uint64)
        co = np.zeros(max(nc.value, 1), np.uint32)
        L.oc_store_copy(h, self.enc_off, self.bit_length, by, self.cp_off, co)
        self.bytes = by[: nb.value]
        self.copied = co[: nc.value]

    def __del__(self):
        try:
            self.cb.o.L.oc_store_free(self.h)
        except Exception:
            pass

    def select(self, hist, k):
        L = self.cb.o.L
        h = np.ascontiguousarray(hist, np.uint64)
        seeds = np.zeros(k, np.uint32)
        marg = np.zeros(k, np.uint64)
        cov = np.zeros(k, np.float64)
        maxd = np.zeros(k, np.uint64)
        padded = L.oc_select_huffman(self.cb.h, self.h, h, h.size, k, seeds, marg, cov, maxd)
        return {"seeds": seeds.tolist(), "marginal": marg.tolist(), "coverage": cov.tolist(), "padded": padded,
                "max_decoded": maxd.tolist()}


def _nz32(a):
    a = np.ascontiguousarray(a, np.uint32)
    return a if a.size else np.zeros(1, np.uint32)


def _nz64(a):
    a = np.ascontiguousarray(a, np.float64)
    return a if a.size else np.zeros(1, np.float64)


class RefLib:
    """The unmodified reference compiled from /root/reference sources (oracle/_ref)."""

    def __init__(self, path: str = REF_PATH):
        if not os.path.exists(path):
            raise RuntimeError(f"reference build missing: {path} (run make -C oracle ref)")
        L = self.L = C.CDLL(path)
        P = C.c_void_p
        _sig(L, "ref_last_error", C.c_char_p, [])
        _sig(L, "ref_graph_new", P, [C.c_uint64, C.c_uint64, u64p, u32p, f64p])
        _sig(L, "ref_graph_load", P, [C.c_char_p])
        _sig(L, "ref_transpose", P, [P])
        _sig(L, "ref_graph_free", None, [P])
        _sig(L, "ref_graph_n", C.c_uint64, [P])
        _sig(L, "ref_graph_m", C.c_uint64, [P])
        _sig(L, "ref_graph_copy", None, [P, u64p, u32p, f64p])
        _sig(L, "ref_sample_block", P, [P, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int])
        _sig(L, "ref_block_total", C.c_uint64, [P])
        _sig(L, "ref_block_copy", None, [P, u64p, u32p])
        _sig(L, "ref_block_free", None, [P])
        _sig(L, "ref_estimate_theta", C.c_int, [P, C.c_uint32, C.c_double, C.c_uint64, C.c_int, u64p,
                                                C.POINTER(C.c_double)])
        _sig(L, "ref_run", P, [P, C.c_uint32, C.c_double, C.c_uint32, C.c_int, C.c_uint64, C.c_int])
        _sig(L, "ref_run_seeds", None, [P, u32p, u64p, f64p, C.POINTER(C.c_uint32)])
        _sig(L, "ref_run_json", C.c_char_p, [P])
        _sig(L, "ref_run_free", None, [P])
        _sig(L, "ref_graph_generate", P, [C.c_int, C.c_uint64, C.c_uint64, C.c_double, C.c_double, C.c_double,
                                          C.c_uint64, C.c_int, C.c_int, C.c_double])
        _sig(L, "ref_probe_block1", P, [P, C.c_uint64, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64])
        _sig(L, "ref_probe_top", C.c_uint32, [P])
        _sig(L, "ref_probe_coded", C.c_uint64, [P])
        _sig(L, "ref_probe_codes", None, [P, u64p, u8p, u64p])
        _sig(L, "ref_probe_enc_sizes", None, [P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)])
        _sig(L, "ref_probe_enc", None, [P, u64p, u8p, u64p, u64p, u32p])
        _sig(L, "ref_probe_block", P, [P])
        _sig(L, "ref_probe_free", None, [P])

    def graph(self, g: CSR):
        return RefGraph(self, self.L.ref_graph_new(g.n, g.m, g.off, _nz32(g.tgt), _nz64(g.prob)))

    def generate(self, gen, weights=("wc", 0.0), reverse: bool = False):
        """A BASELINE-config graph built inside the reference library by oracle/gen_graph.c
        (no Python copy: the c5 graph is 17 GB as immx::Graph).  reverse=False: forward."""
        kind = 0 if gen[0] == "rmat" else 1
        h = self.L.ref_graph_generate(kind, gen[1], gen[2], 0.57, 0.19, 0.19, gen[3], int(reverse),
                                      0 if weights[0] == "wc" else 1, float(weights[1]))
        if not h:
            raise RuntimeError(self.L.ref_last_error().decode())
        return RefGraph(self, h)

    def load(self, path: str):
        h = self.L.ref_graph_load(path.encode())
        if not h:
            raise RuntimeError(self.L.ref_last_error().decode())
        return RefGraph(self, h)


class RefGraph:
    def __init__(self, ref: RefLib, h):
        self.r, self.h = ref, h

    def __del__(self):
        try:
            self.r.L.ref_graph_free(self.h)
        except Exception:
            pass

    @property
    def n(self):
        return self.r.L.ref_graph_n(self.h)

    def transpose(self) -> "RefGraph":
        return RefGraph(self.r, self.r.L.ref_transpose(self.h))

    def csr(self) -> CSR:
        n, m = self.r.L.ref_graph_n(self.h), self.r.L.ref_graph_m(self.h)
        off = np.zeros(n + 1, np.uint64)
        tgt = np.zeros(max(m, 1), np.uint32)
        prob = np.zeros(max(m, 1), np.float64)
        self.r.L.ref_graph_copy(self.h, off, tgt, prob)
        return CSR(n, off, tgt[:m].copy(), prob[:m].copy())

    def sample_block(self, count, first=0, seed=42, workers=1):
        L = self.r.L
        b = L.ref_sample_block(self.h, count, first, seed, workers)
        tot = L.ref_block_total(b)
        offs = np.zeros(count + 1, np.uint64)
        mem = np.zeros(max(tot, 1), np.uint32)
        L.ref_block_copy(b, offs, mem)
        L.ref_block_free(b)
        return offs, mem[:tot].copy()

    def probe_block1(self, per_block, seed, workers, lo, hi):
        """Block 1 of run() through the reference's public functions (ref_shim.cpp
        ref_probe_block1): codebook, block-1 histogram, top, raw and encoded sets [lo, hi)."""
        L = self.r.L
        h = L.ref_probe_block1(self.h, per_block, seed, workers, lo, hi)
        if not h:
            raise RuntimeError(L.ref_last_error().decode())
        try:
            n = self.n
            bits = np.zeros(n, np.uint64)
            lens = np.zeros(n, np.uint8)
            hist = np.zeros(n, np.uint64)
            L.ref_probe_codes(h, bits, lens, hist)
            nb, nc = C.c_uint64(), C.c_uint64()
            L.ref_probe_enc_sizes(h, C.byref(nb), C.byref(nc))
            w = hi - lo
            byte_off = np.zeros(w + 1, np.uint64)
            data = np.zeros(max(nb.value, 1), np.uint8)
            bitlen = np.zeros(max(w, 1), np.uint64)
            cp_off = np.zeros(w + 1, np.uint64)
            copied = np.zeros(max(nc.value, 1), np.uint32)
            L.ref_probe_enc(h, byte_off, data, bitlen, cp_off, copied)
            b = L.ref_probe_block(h)
            tot = L.ref_block_total(b)
            offs = np.zeros(per_block + 1, np.uint64)
            mem = np.zeros(max(tot, 1), np.uint32)
            L.ref_block_copy(b, offs, mem)
            raw_off = offs[lo:hi + 1] - offs[lo]
            raw = mem[int(offs[lo]):int(offs[hi])].copy()
            return {"top": int(L.ref_probe_top(h)), "coded": int(L.ref_probe_coded(h)), "code_bits": bits,
                    "code_len": lens, "hist": hist, "enc_byte_off": byte_off, "enc_bytes": data[:nb.value],
                    "enc_bitlen": bitlen[:w], "enc_cp_off": cp_off, "enc_copied": copied[:nc.value],
                    "raw_off": raw_off, "raw": raw, "block_members": int(tot)}
        finally:
            L.ref_probe_free(h)

    def estimate_theta(self, k, eps, seed=42, workers=1):
        out = np.zeros(3, np.uint64)
        F = C.c_double()
        if self.r.L.ref_estimate_theta(self.h, k, eps, seed, workers, out, C.byref(F)) != 0:
            raise RuntimeError(self.r.L.ref_last_error().decode())
        return {"theta": int(out[0]), "exit_iteration": int(out[1]), "estimation_samples": int(out[2]),
                "covered_fraction": F.value}

    def run(self, k, epsilon=0.5, blocks=8, mode="auto", seed=42, workers=1):
        import json
        L = self.r.L
        h = L.ref_run(self.h, k, epsilon, blocks, -1 if mode == "auto" else MODES[mode], seed, workers)
        if not h:
            raise RuntimeError(L.ref_last_error().decode())
        seeds = np.zeros(k, np.uint32)
        marg = np.zeros(k, np.uint64)
        cov = np.zeros(k, np.float64)
        pad = C.c_uint32()
        L.ref_run_seeds(h, seeds, marg, cov, C.byref(pad))
        stats = json.loads(L.ref_run_json(h).decode())
        L.ref_run_free(h)
        return {"seeds": seeds.tolist(), "marginal": marg.tolist(), "coverage": cov.tolist(),
                "padded": pad.value, "stats": stats}


def load_ref_core():
    """Import the reference's own pybind module (oracle/_ref/immx_ref/_core) if built."""
    import importlib.util
    import glob
    cands = glob.glob(os.path.join(HERE, "_ref", "immx_ref", "_core*.so"))
    if not cands:
        return None
    spec = importlib.util.spec_from_file_location("_core", cands[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod
