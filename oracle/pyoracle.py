"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU oracle and the compiled reference.

* ``Oracle``    — oracle/_build/libspecpar_oracle.so, the C restatement (oracle/specpar_oracle.c).
* ``Reference`` — oracle/_ref/libspecpar_ref.so, the UNMODIFIED reference sources
                  (/root/reference/proj/src) + our C shim (oracle/ref_shim.cpp).  Only present where
                  it was built (oracle/Makefile ``ref`` target); tests skip when absent.

Allowed importers: tests/, __graft_entry__.smoke(), bench.py (cpu_baseline / --impl reference legs).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libspecpar_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspecpar_ref.so")

SOURCES = ["prior", "dynamic", "rejected", "context", "miss"]
ARGMAX_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_int),
                        C.c_int, C.POINTER(C.c_int))
IntP = C.POINTER(C.c_int)
PROBS_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_int),
                       C.c_int, C.POINTER(C.c_double))


def _ints(xs):
    xs = list(xs)
    return (C.c_int * max(1, len(xs)))(*xs)


def build_oracle() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return ORACLE_SO


class OracleError(RuntimeError):
    pass


def make_argmax_callback(fn):
    """Wrap a python ``fn(ctx:list[int], cands:list[int]) -> list[int]`` (|cands|+1 argmax ids)."""

    def cb(_user, ctx, L, cands, c, out):
        try:
            ids = fn([ctx[i] for i in range(L)], [cands[i] for i in range(c)])
            for i, v in enumerate(ids):
                out[i] = int(v)
            return 0
        except Exception:  # noqa: BLE001 — reported through the C status
            import traceback
            traceback.print_exc()
            return -1

    return ARGMAX_FN(cb)


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build_oracle()
        L = C.CDLL(path)
        self.lib = L
        L.orc_last_error.restype = C.c_char_p
        L.orc_table_build.restype = C.c_void_p
        L.orc_table_parse.restype = C.c_void_p
        L.orc_table_serialize.restype = C.c_void_p
        L.orc_table_serialize.argtypes = [C.c_void_p]
        L.orc_table_free.argtypes = [C.c_void_p]
        L.orc_table_vocab.argtypes = [C.c_void_p]
        L.orc_table_argmax_rows.argtypes = [C.c_void_p, IntP, C.c_int, IntP, C.c_int, IntP]
        L.orc_store_new.restype = C.c_void_p
        L.orc_store_free.argtypes = [C.c_void_p]
        L.orc_store_serialize_layer.restype = C.c_void_p
        L.orc_store_serialize_layer.argtypes = [C.c_void_p, C.c_int]
        L.orc_layer_occurrences.restype = C.c_long
        L.orc_layer_occurrences.argtypes = [C.c_void_p, C.c_int]
        L.orc_layer_insert.argtypes = [C.c_void_p, C.c_int, IntP, C.c_int, C.c_long]
        L.orc_store_record.argtypes = [C.c_void_p, C.c_int, IntP, C.c_int]
        L.orc_store_flush.argtypes = [C.c_void_p]
        L.orc_store_set_rejected_enabled.argtypes = [C.c_void_p, C.c_int]
        L.orc_store_lookup.argtypes = [C.c_void_p, IntP, C.c_int, C.c_int, IntP, IntP, IntP, IntP]
        L.orc_store_stats.argtypes = [C.c_void_p, C.POINTER(C.c_long)]
        L.orc_store_load_dstore.argtypes = [C.c_void_p, C.c_int, C.c_char_p]
        L.orc_free.argtypes = [C.c_void_p]
        L.orc_run_config.argtypes = [C.c_char_p, C.c_char_p, IntP, C.c_int, IntP,
                                     C.POINTER(C.c_void_p), C.POINTER(C.c_double)]
        L.orc_run.argtypes = [C.c_int, ARGMAX_FN, C.c_void_p, C.c_int, ARGMAX_FN, C.c_void_p,
                              C.c_void_p, IntP, C.c_int, C.c_int, C.c_void_p, IntP, C.c_int, IntP,
                              C.POINTER(C.c_void_p), C.POINTER(C.c_double)]
        L.orc_run_ar.argtypes = [C.c_int, ARGMAX_FN, C.c_void_p, IntP, C.c_int, C.c_int,
                                 C.c_double, IntP, C.c_int, IntP, C.POINTER(C.c_void_p),
                                 C.POINTER(C.c_double)]
        L.orc_gen_corpus.argtypes = [C.c_int, C.c_double, C.c_int, C.c_uint64, IntP, IntP, IntP]

    def _err(self):
        raise OracleError(self.lib.orc_last_error().decode())

    def _take_str(self, p) -> str:
        s = C.cast(p, C.c_char_p).value.decode()
        self.lib.orc_free(p)
        return s

    # -- corpus / tables ------------------------------------------------------------------
    def gen_corpus(self, vocab, rho, length, seed):
        toks = (C.c_int * length)()
        lens = (C.c_int * (length // 64 + 2))()
        n = C.c_int()
        if self.lib.orc_gen_corpus(vocab, rho, length, seed, toks, lens, C.byref(n)):
            self._err()
        out, at = [], 0
        for i in range(n.value):
            out.append(list(toks[at:at + lens[i]]))
            at += lens[i]
        return out

    def table_build(self, corpus, order, smoothing, vocab) -> "Table":
        flat = [t for s in corpus for t in s]
        h = self.lib.orc_table_build(_ints(flat), _ints(len(s) for s in corpus), len(corpus),
                                     order, C.c_double(smoothing), vocab)
        if not h:
            self._err()
        return Table(self, h)

    def table_parse(self, text: str) -> "Table":
        h = self.lib.orc_table_parse(text.encode())
        if not h:
            self._err()
        return Table(self, h)

    # -- store ----------------------------------------------------------------------------
    def store(self, max_order=3, depth=10) -> "Store":
        return Store(self, self.lib.orc_store_new(max_order, depth))

    # -- loops ----------------------------------------------------------------------------
    def run_config(self, cfg_text: str, method: str | None = None, cap: int = 1 << 16):
        out = (C.c_int * cap)()
        n = C.c_int()
        js = C.c_void_p()
        m = (C.c_double * 8)()
        if self.lib.orc_run_config(cfg_text.encode(), method.encode() if method else None, out,
                                   cap, C.byref(n), C.byref(js), m):
            self._err()
        return list(out[:n.value]), self._take_str(js), list(m)

    def run(self, draft_vocab, draft_cb, target_vocab, target_cb, store: "Store", prompt, max_new,
            gamma=4, depth=10, draft_retrieval=True, target_retrieval=True, t_target=1.0,
            t_draft=0.25, t_lookup=0.0, t_sync=0.0, cap=1 << 16, duser=None, tuser=None):
        class Opts(C.Structure):
            _fields_ = [("gamma", C.c_int), ("depth", C.c_int), ("dr", C.c_int), ("tr", C.c_int),
                        ("t_target", C.c_double), ("t_draft", C.c_double),
                        ("t_lookup", C.c_double), ("t_sync", C.c_double)]
        o = Opts(gamma, depth, int(draft_retrieval), int(target_retrieval), t_target, t_draft,
                 t_lookup, t_sync)
        out = (C.c_int * cap)()
        n = C.c_int()
        js = C.c_void_p()
        m = (C.c_double * 8)()
        if self.lib.orc_run(draft_vocab, draft_cb, duser, target_vocab, target_cb, tuser, store.h,
                            _ints(prompt), len(prompt), max_new, C.byref(o), out, cap, C.byref(n),
                            C.byref(js), m):
            self._err()
        return list(out[:n.value]), self._take_str(js), list(m)

    def run_ar(self, target_vocab, target_cb, prompt, max_new, t_target=1.0, cap=1 << 16):
        out = (C.c_int * cap)()
        n = C.c_int()
        js = C.c_void_p()
        m = (C.c_double * 8)()
        if self.lib.orc_run_ar(target_vocab, target_cb, None, _ints(prompt), len(prompt), max_new,
                               t_target, out, cap, C.byref(n), C.byref(js), m):
            self._err()
        return list(out[:n.value]), self._take_str(js), list(m)


class Table:
    def __init__(self, o: Oracle, h):
        self.o, self.h = o, h

    def __del__(self):
        try:
            self.o.lib.orc_table_free(self.h)
        except Exception:  # noqa: BLE001
            pass

    @property
    def vocab(self):
        return self.o.lib.orc_table_vocab(self.h)

    def serialize(self) -> str:
        return self.o._take_str(self.o.lib.orc_table_serialize(self.h))

    def argmax_rows(self, ctx, cands):
        out = (C.c_int * (len(cands) + 1))()
        if self.o.lib.orc_table_argmax_rows(self.h, _ints(ctx), len(ctx), _ints(cands), len(cands),
                                            out):
            self.o._err()
        return list(out)

    def callback(self):
        lib = self.o.lib
        h = self.h

        def cb(_u, ctx, L, cands, c, out):
            return lib.orc_table_argmax_rows(h, ctx, L, cands, c, out)
        self._cb = ARGMAX_FN(cb)
        return self._cb


class Store:
    def __init__(self, o: Oracle, h):
        self.o, self.h = o, h

    def __del__(self):
        try:
            self.o.lib.orc_store_free(self.h)
        except Exception:  # noqa: BLE001
            pass

    def insert(self, layer: int, toks, step: int):
        if self.o.lib.orc_layer_insert(self.h, layer, _ints(toks), len(toks), step):
            self.o._err()

    def record(self, layer: int, toks):
        if self.o.lib.orc_store_record(self.h, layer, _ints(toks), len(toks)):
            self.o._err()

    def flush(self):
        self.o.lib.orc_store_flush(self.h)

    def set_rejected_enabled(self, on: bool):
        self.o.lib.orc_store_set_rejected_enabled(self.h, int(on))

    def load_dstore(self, layer: int, text: str):
        if self.o.lib.orc_store_load_dstore(self.h, layer, text.encode()):
            self.o._err()

    def serialize(self, layer: int) -> str:
        return self.o._take_str(self.o.lib.orc_store_serialize_layer(self.h, layer))

    def occurrences(self, layer: int) -> int:
        return self.o.lib.orc_layer_occurrences(self.h, layer)

    def lookup(self, ctx, d):
        cands = (C.c_int * max(1, d + len(ctx)))()
        n, src, order = C.c_int(), C.c_int(), C.c_int()
        if self.o.lib.orc_store_lookup(self.h, _ints(ctx), len(ctx), d, cands, C.byref(n),
                                       C.byref(src), C.byref(order)):
            self.o._err()
        return list(cands[:n.value]), SOURCES[src.value], order.value

    def stats(self):
        s = (C.c_long * 6)()
        self.o.lib.orc_store_stats(self.h, s)
        return list(s)


def make_probs_callback(fn, vocab):
    """Wrap ``fn(ctx, cands) -> float64 array (|cands|+1, vocab)`` as the reference's proxy forward."""
    import numpy as np

    def cb(_user, ctx, L, cands, c, out):
        try:
            rows = np.ascontiguousarray(fn([ctx[i] for i in range(L)], [cands[i] for i in range(c)]),
                                        dtype=np.float64)
            assert rows.shape == (c + 1, vocab), rows.shape
            C.memmove(out, rows.ctypes.data, rows.nbytes)
            return 0
        except Exception:  # noqa: BLE001 — reported through the C status
            import traceback
            traceback.print_exc()
            return -1

    return PROBS_FN(cb)


class Reference:
    """The unmodified reference (oracle/_ref).  Raises FileNotFoundError when not built."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        self.lib = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_run_config.argtypes = [C.c_char_p, C.c_char_p, IntP, C.c_int, IntP, C.c_char_p,
                                     C.c_long, C.POINTER(C.c_double)]
        L.ref_export_setup.argtypes = [C.c_char_p, C.c_char_p, C.c_long, C.c_char_p, C.c_long,
                                       C.c_char_p, C.c_long, IntP, IntP, C.c_int]
        L.ref_gen_corpus.argtypes = [C.c_int, C.c_double, C.c_int, C.c_ulonglong, IntP, IntP,
                                     IntP, C.c_int]
        L.ref_lookup_batch.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, IntP, IntP,
                                       C.POINTER(C.c_long), IntP, C.c_int, IntP, IntP, IntP,
                                       C.c_int, IntP, IntP, IntP, IntP, C.POINTER(C.c_long)]
        L.ref_run_callback.argtypes = [C.c_int, ARGMAX_FN, C.c_void_p, ARGMAX_FN, C.c_void_p,
                                       C.c_int, C.c_int, IntP, IntP, IntP, C.c_int, C.c_int,
                                       C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                       C.c_double, C.c_double, C.c_double, IntP, C.c_int, IntP,
                                       C.c_char_p, C.c_long, C.POINTER(C.c_double)]
        L.ref_run_callback_probs.argtypes = [C.c_int, PROBS_FN, C.c_void_p, PROBS_FN, C.c_void_p,
                                             C.c_int, C.c_int, IntP, IntP, IntP, C.c_int, C.c_int,
                                             C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                             C.c_double, C.c_double, C.c_double, C.c_double,
                                             C.c_ulonglong, C.c_char_p, IntP, C.c_int, IntP,
                                             C.c_char_p, C.c_long, C.POINTER(C.c_double)]

    def _err(self):
        raise OracleError(self.lib.ref_last_error().decode())

    def run_config(self, cfg_text: str, method: str, cap: int = 1 << 16, jcap: int = 1 << 24):
        out = (C.c_int * cap)()
        n = C.c_int()
        js = C.create_string_buffer(jcap)
        m = (C.c_double * 8)()
        if self.lib.ref_run_config(cfg_text.encode(), method.encode(), out, cap, C.byref(n), js,
                                   jcap, m):
            self._err()
        return list(out[:n.value]), js.value.decode(), list(m)

    def export_setup(self, cfg_text: str, cap: int = 1 << 25):
        d = C.create_string_buffer(cap)
        t = C.create_string_buffer(cap)
        p = C.create_string_buffer(cap)
        prompt = (C.c_int * 65536)()
        n = C.c_int()
        if self.lib.ref_export_setup(cfg_text.encode(), d, cap, t, cap, p, cap, prompt, C.byref(n),
                                     65536):
            self._err()
        return d.value.decode(), t.value.decode(), p.value.decode(), list(prompt[:n.value])

    def gen_corpus(self, vocab, rho, length, seed):
        toks = (C.c_int * length)()
        lens = (C.c_int * (length // 64 + 2))()
        n = C.c_int()
        if self.lib.ref_gen_corpus(vocab, rho, length, seed, toks, lens, C.byref(n),
                                   length // 64 + 2):
            self._err()
        out, at = [], 0
        for i in range(n.value):
            out.append(list(toks[at:at + lens[i]]))
            at += lens[i]
        return out

    def lookup_batch(self, max_order, inserts, queries, rejected_enabled=True, depth_cfg=10):
        """inserts: [(layer, tokens, step)], queries: [(ctx, d)] -> ([(cands, src, order)], stats)"""
        dcap = max([d for _, d in queries] + [1]) + max([len(c) for c, _ in queries] + [1])
        flat = [t for _, toks, _ in inserts for t in toks]
        steps = (C.c_long * max(1, len(inserts)))(*[s for _, _, s in inserts])
        qflat = [t for c, _ in queries for t in c]
        nq = len(queries)
        oc = (C.c_int * (nq * dcap))()
        on, osrc, oord = (C.c_int * nq)(), (C.c_int * nq)(), (C.c_int * nq)()
        st = (C.c_long * 6)()
        if self.lib.ref_lookup_batch(max_order, depth_cfg, int(rejected_enabled), len(inserts),
                                     _ints(l for l, _, _ in inserts),
                                     _ints(len(t) for _, t, _ in inserts), steps, _ints(flat), nq,
                                     _ints(len(c) for c, _ in queries), _ints(qflat),
                                     _ints(d for _, d in queries), dcap, oc, on, osrc, oord, st):
            self._err()
        res = [(list(oc[q * dcap:q * dcap + on[q]]), SOURCES[osrc[q]], oord[q]) for q in range(nq)]
        return res, list(st)

    def run_callback(self, vocab, draft_cb, target_cb, prior, prompt, max_new, max_order=3,
                     gamma=4, depth=10, draft_retrieval=True, target_retrieval=True,
                     rejected_enabled=True, t_target=1.0, t_draft=0.25, t_lookup=0.0, t_sync=0.0,
                     cap=1 << 16, jcap=1 << 24):
        out = (C.c_int * cap)()
        n = C.c_int()
        js = C.create_string_buffer(jcap)
        m = (C.c_double * 8)()
        flat = [t for s in prior for t in s]
        if self.lib.ref_run_callback(vocab, draft_cb, None, target_cb, None, max_order, len(prior),
                                     _ints(len(s) for s in prior), _ints(flat), _ints(prompt),
                                     len(prompt), max_new, gamma, depth, int(draft_retrieval),
                                     int(target_retrieval), int(rejected_enabled), t_target,
                                     t_draft, t_lookup, t_sync, out, cap, C.byref(n), js, jcap, m):
            self._err()
        return list(out[:n.value]), js.value.decode(), list(m)


def _run_callback_probs(self, vocab, draft_cb, target_cb, prior, prompt, max_new, temperature, seed,
                        method="double", max_order=3, gamma=4, depth=10, draft_retrieval=True,
                        target_retrieval=True, rejected_enabled=True, t_target=1.0, t_draft=0.25,
                        t_lookup=0.0, t_sync=0.0, cap=1 << 16, jcap=1 << 24):
    """The reference loop at temperature > 0 over callback distributions (ref_run_callback_probs)."""
    out = (C.c_int * cap)()
    n = C.c_int()
    js = C.create_string_buffer(jcap)
    m = (C.c_double * 8)()
    flat = [t for s in prior for t in s]
    if self.lib.ref_run_callback_probs(vocab, draft_cb, None, target_cb, None, max_order, len(prior),
                                       _ints(len(s) for s in prior), _ints(flat), _ints(prompt),
                                       len(prompt), max_new, gamma, depth, int(draft_retrieval),
                                       int(target_retrieval), int(rejected_enabled), t_target, t_draft,
                                       t_lookup, t_sync, float(temperature), int(seed), method.encode(),
                                       out, cap, C.byref(n), js, jcap, m):
        self._err()
    return list(out[:n.value]), js.value.decode(), list(m)


Reference.run_callback_probs = _run_callback_probs


def reference_or_none():
    try:
        return Reference()
    except (FileNotFoundError, OSError):
        return None


# --------------------------------------------------------------------------- verifier (T >= 0)
class OracleInvalidArgument(OracleError):  # std::invalid_argument
    pass


class OracleRuntimeError(OracleError):  # std::runtime_error
    pass


def _rows(rows):
    rows = [list(map(float, r)) for r in (rows or [])]
    off = [0]
    for r in rows:
        off.append(off[-1] + len(r))
    flat = [x for r in rows for x in r]
    return (C.c_double * max(1, len(flat)))(*flat), (C.c_long * len(off))(*off), len(rows)


def _dbl(xs):
    xs = [float(x) for x in xs]
    return (C.c_double * max(1, len(xs)))(*xs)


def _splitmix64(x: int) -> int:  # rng.hpp:8-13
    M = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & M
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
    x = ((x ^ (x >> 27)) * 0x94D49BB133111EB) & M  # the reference's constant (rng.hpp:11)
    return x ^ (x >> 31)


class _MT64(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_int)]


class _VerifierCalls:
    """The five verifier functions over either checker; `rng` objects come from .rng()/.derive_rng()."""

    def _call(self, rc):
        if rc == -1:
            raise OracleInvalidArgument(self._msg())
        if rc != 0:
            raise OracleRuntimeError(self._msg())

    def accept_prob(self, p, q, x):
        out = C.c_double()
        self._call(self._f["accept"](_dbl(p), len(p), _dbl(q), len(q), x, C.byref(out)))
        return out.value

    def residual_sample(self, p, q, rng):
        out = C.c_int()
        self._call(self._f["residual"](_dbl(p), len(p), _dbl(q), len(q), self._rp(rng), C.byref(out)))
        return out.value

    def residual_sample_point_mass(self, p, x, rng):
        out = C.c_int()
        self._call(self._f["point"](_dbl(p), len(p), x, self._rp(rng), C.byref(out)))
        return out.value

    def verify_against_target(self, draft, draft_probs, target_probs, temperature, rng):
        dp, doff, nd = _rows(draft_probs)
        tp, toff, nt = _rows(target_probs)
        out = C.c_int()
        self._call(self._f["verify"](_ints(draft), len(draft), dp, doff, nd, tp, toff, nt, float(temperature),
                                     self._rp(rng), C.byref(out)))
        return None if out.value < 0 else out.value

    def guided_output(self, draft, draft_probs, guide_tokens, guide_probs, first_reject, temperature, rng):
        dp, doff, nd = _rows(draft_probs)
        gp, goff, ng = _rows(guide_probs)
        cap = len(draft) + len(guide_tokens) + 1
        out = (C.c_int * cap)()
        n, acc, kind = C.c_int(), C.c_int(), C.c_int()
        self._call(self._f["guided"](_ints(draft), len(draft), dp, doff, nd, _ints(guide_tokens), len(guide_tokens),
                                     gp, goff, ng, -1 if first_reject is None else int(first_reject),
                                     float(temperature), self._rp(rng), out, cap, C.byref(n), C.byref(acc),
                                     C.byref(kind)))
        return acc.value, list(out[:n.value]), ["all_accepted", "correction", "extension",
                                                "residual_correction"][kind.value]


class OracleVerifier(_VerifierCalls):
    def __init__(self, oracle: Oracle):
        L = oracle.lib
        self._msg = lambda: L.orc_last_error().decode()
        rows = [C.c_void_p, C.POINTER(C.c_long), C.c_int]
        dbl = [C.POINTER(C.c_double), C.c_int]
        L.orc_mt64_seed.argtypes = [C.POINTER(_MT64), C.c_uint64]
        L.orc_uniform.restype = C.c_double
        L.orc_uniform.argtypes = [C.POINTER(_MT64)]
        L.orc_accept_prob.argtypes = dbl + dbl + [C.c_int, C.POINTER(C.c_double)]
        L.orc_residual_sample.argtypes = dbl + dbl + [C.POINTER(_MT64), IntP]
        L.orc_residual_point_mass.argtypes = dbl + [C.c_int, C.POINTER(_MT64), IntP]
        L.orc_verify_against_target.argtypes = [IntP, C.c_int] + rows + rows + [C.c_double, C.POINTER(_MT64), IntP]
        L.orc_guided_output.argtypes = ([IntP, C.c_int] + rows + [IntP, C.c_int] + rows +
                                        [C.c_int, C.c_double, C.POINTER(_MT64), IntP, C.c_int, IntP, IntP, IntP])
        self._f = {"accept": L.orc_accept_prob, "residual": L.orc_residual_sample,
                   "point": L.orc_residual_point_mass, "verify": L.orc_verify_against_target,
                   "guided": L.orc_guided_output}
        self._L = L
        self._rp = lambda r: C.byref(r)

    def rng(self, seed: int):  # Rng(seed)
        g = _MT64()
        self._L.orc_mt64_seed(C.byref(g), C.c_uint64(seed))
        return g

    def derive_rng(self, seed: int, round_: int, lane: int):  # rng.hpp:33-35
        M = (1 << 64) - 1
        return self.rng(_splitmix64((seed ^ _splitmix64((round_ * 4 + lane + 1) & M)) & M))

    def uniform(self, g):
        return self._L.orc_uniform(C.byref(g))


class ReferenceVerifier(_VerifierCalls):
    def __init__(self, ref: "Reference"):
        L = ref.lib
        self._msg = lambda: L.ref_last_error().decode()
        rows = [C.c_void_p, C.POINTER(C.c_long), C.c_int]
        dbl = [C.POINTER(C.c_double), C.c_int]
        L.ref_rng_new.restype = C.c_void_p
        L.ref_rng_new.argtypes = [C.c_ulonglong]
        L.ref_rng_derive.restype = C.c_void_p
        L.ref_rng_derive.argtypes = [C.c_ulonglong, C.c_ulonglong, C.c_ulonglong]
        L.ref_rng_free.argtypes = [C.c_void_p]
        L.ref_rng_uniform.restype = C.c_double
        L.ref_rng_uniform.argtypes = [C.c_void_p]
        L.ref_accept_prob.argtypes = dbl + dbl + [C.c_int, C.POINTER(C.c_double)]
        L.ref_residual_sample.argtypes = dbl + dbl + [C.c_void_p, IntP]
        L.ref_residual_point_mass.argtypes = dbl + [C.c_int, C.c_void_p, IntP]
        L.ref_verify_against_target.argtypes = [IntP, C.c_int] + rows + rows + [C.c_double, C.c_void_p, IntP]
        L.ref_guided_output.argtypes = ([IntP, C.c_int] + rows + [IntP, C.c_int] + rows +
                                        [C.c_int, C.c_double, C.c_void_p, IntP, C.c_int, IntP, IntP, IntP])
        self._f = {"accept": L.ref_accept_prob, "residual": L.ref_residual_sample,
                   "point": L.ref_residual_point_mass, "verify": L.ref_verify_against_target,
                   "guided": L.ref_guided_output}
        self._L = L
        self._rp = lambda r: r.h

    class _Rng:
        def __init__(self, L, h):
            self.L, self.h = L, C.c_void_p(h)

        def __del__(self):
            self.L.ref_rng_free(self.h)

    def rng(self, seed: int):
        return self._Rng(self._L, self._L.ref_rng_new(seed))

    def derive_rng(self, seed: int, round_: int, lane: int):
        return self._Rng(self._L, self._L.ref_rng_derive(seed, round_, lane))

    def uniform(self, g):
        return self._L.ref_rng_uniform(g.h)
