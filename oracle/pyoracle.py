"""ctypes bindings for the test-infrastructure oracles (TEST INFRASTRUCTURE ONLY).

Two libraries with identical C signatures:

* ``oracle/liborc.so``          -- the plain-C restatement (``orc_*``), always built.
* ``oracle/_ref/libhh_ref.so``  -- the unmodified reference headers compiled in
  place (``ref_*``); present when built in a container that has
  ``/root/reference`` (the prebuilt .so travels to the GPU box).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may
import this module.  The product package never does.

All numpy arrays are converted to contiguous float64/float32/int64 buffers.
Error codes: -1 <-> std::invalid_argument, -2 <-> std::logic_error.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORC_PATH = HERE / "liborc.so"
REF_PATH = HERE / "_ref" / "libhh_ref.so"

EINVAL = -1
ESTATE = -2

KIND = {"topk": 0, "topp": 1, "threshold": 2, "ratio": 3}


class OracleError(RuntimeError):
    pass


class InvalidArgument(OracleError, ValueError):
    """Mirrors std::invalid_argument."""


class LogicError(OracleError):
    """Mirrors std::logic_error."""


def _check(rc):
    if rc == EINVAL:
        raise InvalidArgument("invalid argument")
    if rc == ESTATE:
        raise LogicError("logic error")
    if rc < 0:
        raise OracleError(f"oracle error {rc}")
    return rc


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


class Oracle:
    """One of the two oracle libraries (prefix 'orc' or 'ref')."""

    def __init__(self, path: Path, prefix: str):
        self.path = Path(path)
        self.prefix = prefix
        self.lib = C.CDLL(str(self.path))
        vp, i64, dbl, flt, i32 = C.c_void_p, C.c_int64, C.c_double, C.c_float, C.c_int
        sig = {
            "dense_attention_f64": (C.c_int, [vp, vp, vp, i64, i64, dbl, vp, vp]),
            "sparse_attention_f64": (C.c_int, [vp, vp, vp, i64, i64, dbl, vp, i64, vp]),
            "args_top_k_f64": (i64, [vp, i64, i64, vp]),
            "args_top_k_f32": (i64, [vp, i64, i64, vp]),
            "gqa_pool_queries_f64": (C.c_int, [vp, i64, i64, i64, vp]),
            "fraction_budget": (i64, [dbl, i64]),
            "select_tokens": (i64, [i32, i64, dbl, vp, i64, vp]),
            "plan_splits": (i64, [i64, i64, vp, i64, vp, vp, vp, i64]),
            "latency_model": (C.c_int, [i64, i64, vp, i64, i64, vp, vp]),
            "decode_step_f64": (
                C.c_int,
                [i64, i64, i64, i64, i64, i64, dbl, vp, vp, vp, vp, i32, i64, dbl, vp, vp, i64,
                 vp, vp, vp],
            ),
        }
        for name, (res, args) in sig.items():
            fn = getattr(self.lib, f"{prefix}_{name}")
            fn.restype, fn.argtypes = res, args
        run_args = [i64, i64, i64, i64, i64, i64, None, vp, vp, vp, vp, vp, i64, vp, vp]
        for sfx, sc in (("f32", flt), ("f64", dbl)):
            fn = getattr(self.lib, f"{prefix}_kernel_run_{sfx}")
            a = list(run_args)
            a[6] = sc
            if prefix == "ref":
                a.append(i64)  # n_workers
            fn.restype, fn.argtypes = C.c_int, a
        if prefix == "ref":
            fn = self.lib.ref_kernel_run_time_f32
            fn.restype = C.c_int
            fn.argtypes = [i64, i64, i64, i64, i64, i64, flt, vp, vp, vp, vp, vp, i64, i64, i64,
                           vp, vp]
        if prefix == "ref":
            self.lib.ref_step_ctx_create.restype = vp
            self.lib.ref_step_ctx_create.argtypes = [i64, i64, i64, i64, flt, vp, vp, vp]
            self.lib.ref_step_ctx_destroy.restype = None
            self.lib.ref_step_ctx_destroy.argtypes = [vp]
            self.lib.ref_step_run.restype = C.c_int
            self.lib.ref_step_run.argtypes = [vp, i64, vp, vp, vp, i64, i64, i64, vp, vp]
        if prefix == "orc":
            self.lib.orc_decode_layer_f32in.restype = C.c_int
            self.lib.orc_decode_layer_f32in.argtypes = [
                i64, i64, i64, i64, i64, dbl, i32, vp, vp, vp, vp, i32, i64, dbl, vp, vp, i64, vp,
                vp, i32]
            self.lib.orc_block_select_f64.restype = i64
            self.lib.orc_block_select_f64.argtypes = [vp, vp, i64, i64, dbl, i64, i64, vp]
            self.lib.orc_pooled_scores_f64.restype = None
            self.lib.orc_pooled_scores_f64.argtypes = [vp, vp, i64, i64, dbl, vp]

    def _fn(self, name):
        return getattr(self.lib, f"{self.prefix}_{name}")

    # ---- attention.hpp -------------------------------------------------
    def dense_attention(self, q, K, V, scale):
        """attention.hpp:50-75 -> (out[d], weights[n])."""
        q, K, V = _f64(q), _f64(K), _f64(V)
        n = K.shape[0] if K.ndim == 2 else 0
        d = q.shape[0]
        out = np.zeros(d)
        w = np.zeros(max(n, 1))
        _check(self._fn("dense_attention_f64")(_p(q), _p(K), _p(V), n, d, scale, _p(out), _p(w)))
        return out, w[:n]

    def sparse_attention(self, q, K, V, scale, idx):
        """attention.hpp:79-104."""
        q, K, V, idx = _f64(q), _f64(K), _f64(V), _i64(idx)
        out = np.zeros(q.shape[0])
        _check(self._fn("sparse_attention_f64")(_p(q), _p(K), _p(V), K.shape[0], q.shape[0],
                                                scale, _p(idx), idx.shape[0], _p(out)))
        return out

    def args_top_k(self, w, k):
        """attention.hpp:108-123 (f64 or f32 by input dtype)."""
        w = np.asarray(w)
        if w.dtype == np.float32:
            w, fn = _f32(w), self._fn("args_top_k_f32")
        else:
            w, fn = _f64(w), self._fn("args_top_k_f64")
        out = np.zeros(max(min(k, w.shape[0]), 1), dtype=np.int64)
        n = _check(fn(_p(w), w.shape[0], k, _p(out)))
        return out[:n]

    def gqa_pool_queries(self, q, group):
        """attention.hpp:127-146.  q: [n_heads][d]."""
        q = _f64(q)
        n, d = q.shape
        out = np.zeros(((n // group) if group > 0 and n % group == 0 else 1, d))
        _check(self._fn("gqa_pool_queries_f64")(_p(q), n, d, group, _p(out)))
        return out

    # ---- policy.hpp ----------------------------------------------------
    def fraction_budget(self, frac, n):
        return int(self._fn("fraction_budget")(frac, n))

    def select_tokens(self, kind, w, k=1, value=0.0):
        """policy.hpp:64-104.  kind in {'topk','topp','threshold','ratio'}."""
        w = _f64(w)
        out = np.zeros(max(w.shape[0], 1), dtype=np.int64)
        n = _check(self._fn("select_tokens")(KIND[kind], k, value, _p(w), w.shape[0], _p(out)))
        return out[:n]

    # ---- kernel_sim.hpp ------------------------------------------------
    def plan_splits(self, head_blocks, num_splits):
        """kernel_sim.hpp:63-110.  head_blocks: [B][H] list sizes.

        Returns (units[n][6] = (b, s, g, begin, end, head_local_split),
        split_blocks[B][S], head_split_count[B][H])."""
        hb = _i64(head_blocks)
        B, H = hb.shape
        sb = np.zeros((B, max(num_splits, 1)), dtype=np.int64)
        hsc = np.zeros((B, H), dtype=np.int64)
        n = _check(self._fn("plan_splits")(B, H, _p(hb), num_splits, _p(sb), _p(hsc), None, 0))
        units = np.zeros((max(n, 1), 6), dtype=np.int64)
        _check(self._fn("plan_splits")(B, H, _p(hb), num_splits, _p(sb), _p(hsc), _p(units), n))
        return units[:n], sb, hsc

    def latency_model(self, head_blocks, num_splits, bytes_per_block):
        """kernel_sim.hpp:284-316 -> dict."""
        hb = _i64(head_blocks)
        B, H = hb.shape
        o = np.zeros(6, dtype=np.int64)
        do = np.zeros(2)
        _check(self._fn("latency_model")(B, H, _p(hb), num_splits, bytes_per_block, _p(o), _p(do)))
        keys = ["total_blocks", "pooled_critical_blocks", "naive_critical_blocks",
                "bytes_per_block", "pooled_critical_bytes", "naive_critical_bytes"]
        r = {k: int(v) for k, v in zip(keys, o)}
        r["mean_split_blocks"], r["balance_ratio"] = float(do[0]), float(do[1])
        return r

    def kernel_run(self, K, V, Q, blocks, *, batch, group, seq_len, block_size=64, scale=1.0,
                   num_splits=1, dtype=np.float32, n_workers=1, exec_counts=False):
        """kernel_sim.hpp:237-279 run<T>.

        K, V: [B*H][seq][d]; Q: [B*Hq][d]; blocks: list (len B*H) of ascending
        block-id lists.  Returns outputs [B*Hq][d] (and exec counts [B*H][nb])."""
        cv = _f32 if dtype == np.float32 else _f64
        sfx = "f32" if dtype == np.float32 else "f64"
        K, V, Q = cv(K), cv(V), cv(Q)
        BH, _, d = K.shape
        group = int(group)
        off = np.zeros(len(blocks) + 1, dtype=np.int64)
        for i, b in enumerate(blocks):
            off[i + 1] = off[i] + len(b)
        ids = _i64(np.concatenate([np.asarray(b, dtype=np.int64) for b in blocks])
                   if off[-1] > 0 else np.zeros(1, dtype=np.int64))
        n_kv_per_b = BH // batch
        nb = (seq_len + block_size - 1) // block_size
        out = np.zeros((Q.shape[0], d), dtype=dtype)
        ec = np.zeros((BH, nb), dtype=np.int64) if exec_counts else None
        args = [batch, n_kv_per_b, group, d, seq_len, block_size, scale, _p(K), _p(V), _p(Q),
                _p(off), _p(ids), num_splits, _p(out), _p(ec)]
        if self.prefix == "ref":
            args.append(n_workers)
        _check(self._fn(f"kernel_run_{sfx}")(*args))
        return (out, ec) if exec_counts else out

    def kernel_run_time(self, K, V, Q, blocks, *, batch, group, seq_len, block_size=64, scale=1.0,
                        num_splits=1, n_workers=1, reps=1):
        """ref only: best wall seconds of hh::kernel::run<float> over reps."""
        K, V, Q = _f32(K), _f32(V), _f32(Q)
        BH, _, d = K.shape
        off = np.zeros(len(blocks) + 1, dtype=np.int64)
        for i, b in enumerate(blocks):
            off[i + 1] = off[i] + len(b)
        ids = _i64(np.concatenate([np.asarray(b, dtype=np.int64) for b in blocks]))
        out = np.zeros((Q.shape[0], d), dtype=np.float32)
        best = np.zeros(1)
        _check(self.lib.ref_kernel_run_time_f32(batch, BH // batch, group, d, seq_len,
                                                block_size, scale, _p(K), _p(V), _p(Q), _p(off),
                                                _p(ids), num_splits, n_workers, reps, _p(out),
                                                _p(best)))
        return float(best[0]), out

    def step_context(self, K, V, Q, *, group, scale):
        """ref only: a reusable whole-step timing context (ref_step_run)."""
        return RefStep(self, K, V, Q, group=group, scale=scale)

    # ---- decode_engine.hpp ---------------------------------------------
    def decode_step(self, q, K, V, roles, *, seq, scale, kind="topk", k=1, value=0.0,
                    sets=None, set_cap=None, trace=False):
        """decode_engine.hpp:109-151 over synthetic inputs (one sequence).

        q: [L][Hq][d]; K, V: [L][H][seq_cap][d]; roles: [L][H] (0=R, 1=S).
        sets: optional list of H index arrays (the engine's sets_).
        Returns dict(out=[L][Hq][d], sets=list, trace=list[L][H] or None)."""
        q, K, V = _f64(q), _f64(K), _f64(V)
        L, H, seq_cap, d = K.shape
        Hq = q.shape[1]
        group = Hq // H
        roles = np.ascontiguousarray(roles, dtype=np.uint8)
        if set_cap is None:
            set_cap = seq
        s_arr = np.zeros((H, set_cap), dtype=np.int64)
        s_len = np.zeros(H, dtype=np.int64)
        if sets is not None:
            for g, s in enumerate(sets):
                s_arr[g, : len(s)] = s
                s_len[g] = len(s)
        out = np.zeros((L, Hq, d))
        tr = np.zeros((L, H, set_cap), dtype=np.int64) if trace else None
        tl = np.zeros((L, H), dtype=np.int64) if trace else None
        _check(self._fn("decode_step_f64")(L, H, group, d, seq, seq_cap, scale, _p(q), _p(K),
                                           _p(V), _p(roles), KIND[kind], k, value, _p(s_arr),
                                           _p(s_len), set_cap, _p(out), _p(tr), _p(tl)))
        res = {"out": out, "sets": [s_arr[g, : s_len[g]].copy() for g in range(H)], "trace": None}
        if trace:
            res["trace"] = [[tr[l, g, : tl[l, g]].copy() for g in range(H)] for l in range(L)]
        return res

    def decode_layer(self, q_l, K_l, V_l, roles_l, state, *, layer0, seq, scale, kind="topk",
                     k=1, value=0.0, pooled_scores=False, threads=0):
        """orc only: one layer of decode_engine.hpp:109-151 for one sequence on
        f32-held inputs (exact upcast to f64; orc_decode_layer_f32in).

        q_l [Hq][d]; K_l, V_l [H][row_stride][d] (f32, rows >= seq ignored);
        roles_l [H]; state: LayerState (the engine's sets_, carried across
        layers).  Returns (out [Hq][d] f64, pooled scores [H][seq] or None)."""
        q_l, K_l, V_l = _f32(q_l), _f32(K_l), _f32(V_l)
        H, row_stride, d = K_l.shape
        Hq = q_l.shape[0]
        roles_l = np.ascontiguousarray(roles_l, dtype=np.uint8)
        out = np.zeros((Hq, d))
        ps = np.zeros((H, seq)) if pooled_scores else None
        th = threads or min(H, os.cpu_count() or 1)
        _check(self.lib.orc_decode_layer_f32in(H, Hq // H, d, seq, row_stride, scale, int(layer0),
                                               _p(roles_l), _p(q_l), _p(K_l), _p(V_l), KIND[kind],
                                               k, value, _p(state.sets), _p(state.len),
                                               state.cap, _p(out), _p(ps), th))
        return out, ps

    # ---- composition oracles (orc only) --------------------------------
    def block_select(self, pooled_q, Kg, seq, scale, block_size, nblk):
        pooled_q, Kg = _f64(pooled_q), _f64(Kg)
        d = pooled_q.shape[0]
        nb = (seq + block_size - 1) // block_size
        out = np.zeros(max(min(nblk, nb), 1), dtype=np.int64)
        n = _check(self.lib.orc_block_select_f64(_p(pooled_q), _p(Kg), seq, d, scale, block_size,
                                                 nblk, _p(out)))
        return out[:n]

    def pooled_scores(self, pooled_q, Kg, seq, scale):
        pooled_q, Kg = _f64(pooled_q), _f64(Kg)
        s = np.zeros(seq)
        self.lib.orc_pooled_scores_f64(_p(pooled_q), _p(Kg), seq, pooled_q.shape[0], scale, _p(s))
        return s


class LayerState:
    """The engine's per-KV-head sets_ (decode_engine.hpp:251) for
    Oracle.decode_layer: sets [H][cap] int64 + lengths [H]."""

    def __init__(self, H, cap):
        self.cap = int(cap)
        self.sets = np.zeros((H, max(self.cap, 1)), dtype=np.int64)
        self.len = np.zeros(H, dtype=np.int64)

    def set(self, g):
        return self.sets[g, : self.len[g]].copy()


class RefStep:
    """One decode step of the reference CPU path, every layer executed
    (oracle/ref_shim.cpp ref_step_run): per layer hh::kernel::run<float> over
    the layer's block lists, then the f64 selection pass of each retrieval
    head.  K, V: [H][L][d] f32 (one layer's caches, reused for every layer);
    Q: [H*G][d]."""

    def __init__(self, o: "Oracle", K, V, Q, *, group, scale):
        self._o = o
        self.K, self.V, self.Q = _f32(K), _f32(V), _f32(Q)
        H, L, d = self.K.shape
        self.H, self.L, self.d = H, L, d
        self.h = o.lib.ref_step_ctx_create(H, group, d, L, scale, _p(self.K), _p(self.V),
                                           _p(self.Q))

    def run(self, roles, blocks, *, num_splits, n_workers, top_k):
        """roles [NL][H]; blocks[l][g] = ascending block ids.  -> (seconds,
        attention seconds, selection seconds)."""
        roles = np.ascontiguousarray(roles, dtype=np.uint8)
        NL = roles.shape[0]
        off = np.zeros((NL, self.H + 1), dtype=np.int64)
        flat = []
        n = 0
        for l in range(NL):
            for g in range(self.H):
                off[l, g] = n
                flat.append(np.asarray(blocks[l][g], dtype=np.int64))
                n += len(blocks[l][g])
            off[l, self.H] = n
        ids = _i64(np.concatenate(flat) if n else np.zeros(1, dtype=np.int64))
        sec = np.zeros(1)
        parts = np.zeros(2)
        _check(self._o.lib.ref_step_run(self.h, NL, _p(roles), _p(off), _p(ids), num_splits,
                                        n_workers, top_k, _p(sec), _p(parts)))
        return float(sec[0]), float(parts[0]), float(parts[1])

    def close(self):
        if self.h:
            self._o.lib.ref_step_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_cache: dict = {}


def orc() -> Oracle:
    """The C restatement (always available once oracle/ is built)."""
    if "orc" not in _cache:
        if not ORC_PATH.exists():
            build()
        _cache["orc"] = Oracle(ORC_PATH, "orc")
    return _cache["orc"]


def ref() -> Oracle | None:
    """The reference itself (None when oracle/_ref was never built)."""
    if "ref" not in _cache:
        _cache["ref"] = Oracle(REF_PATH, "ref") if REF_PATH.exists() else None
    return _cache["ref"]


def build() -> None:
    """make -C oracle (C restatement; _ref too when /root/reference is present)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", str(HERE)], check=True,
                   env={**os.environ})
