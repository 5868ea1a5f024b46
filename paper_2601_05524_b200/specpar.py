"""Python mirror of the reference's ``specpar`` decode-path API (proj/include/specpar/*.hpp), backed by
the B200 C-ABI (include/double_b200.h).  Same names, argument meaning and error types:

=========================================  =====================================================
reference (C++)                            here
=========================================  =====================================================
HierarchicalDatastore(n, d)                HierarchicalDatastore(n, d, device=0)
  .prior/.dynamic/.rejected .insert(s, k)    .prior/.dynamic/.rejected .insert(s, k)
  .lookup(ctx, d) -> LookupResult            .lookup(ctx, d) -> LookupResult
  .record_accepted / .record_rejected        same
  .flush_session(), .rejected_enabled        same; .stats -> LookupStats
build_prior(corpora, N, K)                 build_prior(store, corpora, K)   (fills store.prior)
TableModel + forward_batch / argmax_token  TableModel.from_model_v1(text) ; forward_batch(m, ctx, c)
run(draft, target, store, prompt, n, opts) run(draft, target, store, prompt, n, opts)
run_vanilla_ar / run_serial_sd (harness)   run_vanilla_ar / run_serial_sd
=========================================  =====================================================

std::invalid_argument -> InvalidArgument (a ValueError), std::runtime_error -> DoubleError,
std::logic_error -> LogicError.  Nothing here computes on the CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._capi import (DoubleError, InvalidArgument, LogicError, PipelineOptions as _Opts, RunMetrics,
                    TransformerConfig, check, lib)

SOURCES = ["prior", "dynamic", "rejected", "context", "miss"]
PRIOR, DYNAMIC, REJECTED = 0, 1, 2

__all__ = ["set_exact_sampling", "NGramIndex", "HierarchicalDatastore", "LookupResult", "LookupStats", "TableModel", "Transformer", "TpTransformer",
           "PipelineOptions", "RunResult", "forward_batch", "forward_logits", "forward_dists", "run",
           "run_vanilla_ar", "run_vanilla_ar_batch", "run_batch", "link_tp_processes",
           "run_serial_sd", "build_prior", "last_run_log", "DoubleError", "InvalidArgument", "LogicError",
           "parse_model_v1", "parse_dstore_v1", "serialize_model", "serialize_index", "save_model",
           "load_model", "save_index", "load_index"]


def _i32(xs) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(list(xs) if not isinstance(xs, np.ndarray) else xs,
                                           dtype=np.int32).reshape(-1))


def _p32(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


@dataclass
class LookupResult:  # datastore.hpp:33-37
    candidates: list
    source: str = "miss"
    matched_order: int = 0


@dataclass
class LookupStats:  # datastore.hpp:39-67
    lookups: int = 0
    prior_hits: int = 0
    dynamic_hits: int = 0
    rejected_hits: int = 0
    fallback_hits: int = 0
    misses: int = 0

    def hits(self):
        return self.prior_hits + self.dynamic_hits + self.rejected_hits + self.fallback_hits

    def hit_rate(self):
        return 0.0 if self.lookups == 0 else self.hits() / self.lookups


class _Layer:
    """One NGramIndex layer of a device store (datastore.hpp:19-27)."""

    def __init__(self, store: "HierarchicalDatastore", layer: int):
        self._s, self._l = store, layer

    def insert(self, tokens, step: int):  # NGramIndex::insert, datastore.cpp:9-20
        a = _i32(tokens)
        check(lib().dbl_store_insert(self._s._h, self._l, _p32(a), len(a), int(step)))

    def clear(self):
        check(lib().dbl_store_clear_layer(self._s._h, self._l))

    def build_index(self):
        """Device n-gram index over the layer's current sequences (lookups unchanged, scans avoided)."""
        check(lib().dbl_store_build_index(self._s._h, self._l))

    @property
    def index_entries(self) -> int:
        v = C.c_int64()
        check(lib().dbl_store_index_entries(self._s._h, self._l, C.byref(v)))
        return v.value

    def _info(self):
        n_s, n_t, occ = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().dbl_store_layer_info(self._s._h, self._l, C.byref(n_s), C.byref(n_t),
                                         C.byref(occ)))
        return n_s.value, n_t.value, occ.value

    def occurrence_count(self) -> int:
        return self._info()[2]

    @property
    def max_order(self):
        return self._s._orders[self._l]

    @max_order.setter
    def max_order(self, v):
        check(lib().dbl_store_set_layer_order(self._s._h, self._l, int(v)))
        self._s._orders[self._l] = int(v)

    def read(self):
        """(sequences, steps) copied back from HBM."""
        n_s, n_t, _ = self._info()
        toks = np.zeros(max(n_t, 1), np.int32)
        lens = np.zeros(max(n_s, 1), np.int32)
        steps = np.zeros(max(n_s, 1), np.int64)
        check(lib().dbl_store_layer_read(self._s._h, self._l, _p32(toks), len(toks), _p32(lens),
                                         steps.ctypes.data_as(C.POINTER(C.c_int64)), len(lens)))
        out, at = [], 0
        for i in range(n_s):
            out.append(toks[at:at + lens[i]].tolist())
            at += lens[i]
        return out, steps[:n_s].tolist()

    @property
    def sequences(self):
        return self.read()[0]


class HierarchicalDatastore:
    """Device-resident three-layer n-gram store (datastore.hpp:72-95)."""

    def __init__(self, n: int = 3, d: int = 10, device: int = 0):
        h = C.c_void_p()
        check(lib().dbl_store_create(int(n), int(d), int(device), C.byref(h)))
        self._h = h
        self.max_order, self.depth, self.device = n, d, device
        self._orders = [n, n, n]
        self._rej = True
        self._layers = (_Layer(self, 0), _Layer(self, 1), _Layer(self, 2))

    # the three NGramIndex layers; assigning a host NGramIndex (e.g. build_prior's) loads it in one upload
    def _set_layer(self, layer: int, idx: "NGramIndex"):
        if not isinstance(idx, NGramIndex):
            raise InvalidArgument("a datastore layer can only be assigned an NGramIndex")
        if layer == PRIOR and idx.steps == list(range(len(idx.sequences))):
            flat, off = _flatten(idx.sequences)
            check(lib().dbl_build_prior(self._h, _i64(off), _p32(flat), len(idx.sequences), int(idx.max_order),
                                        len(idx.sequences)))
            self._orders[layer] = int(idx.max_order)
            return
        L = self._layers[layer]
        L.clear()
        L.max_order = idx.max_order
        for seq, step in zip(idx.sequences, idx.steps):
            L.insert(seq, step)

    prior = property(lambda self: self._layers[0], lambda self, v: self._set_layer(0, v))
    dynamic = property(lambda self: self._layers[1], lambda self, v: self._set_layer(1, v))
    rejected = property(lambda self: self._layers[2], lambda self, v: self._set_layer(2, v))

    def copy(self) -> "HierarchicalDatastore":
        """A deep copy on the device (the reference's store is a value type, test_pipeline.cpp:170-187)."""
        h = C.c_void_p()
        check(lib().dbl_store_clone(self._h, C.byref(h)))
        c = HierarchicalDatastore.__new__(HierarchicalDatastore)
        c._h = h
        c.max_order, c.depth, c.device = self.max_order, self.depth, self.device
        c._orders = list(self._orders)
        c._rej = self._rej
        c._layers = (_Layer(c, 0), _Layer(c, 1), _Layer(c, 2))
        return c

    __copy__ = copy

    def __deepcopy__(self, memo):
        return self.copy()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().dbl_store_destroy(h)
            self._h = None

    @property
    def rejected_enabled(self) -> bool:
        return self._rej

    @rejected_enabled.setter
    def rejected_enabled(self, on: bool):
        check(lib().dbl_store_set_rejected_enabled(self._h, int(bool(on))))
        self._rej = bool(on)

    @property
    def step_counter(self) -> int:
        v = C.c_int64()
        check(lib().dbl_store_get_step(self._h, C.byref(v)))
        return v.value

    @step_counter.setter
    def step_counter(self, v: int):
        check(lib().dbl_store_set_step(self._h, int(v)))

    def lookup(self, context, d: int) -> LookupResult:  # datastore.cpp:82-132
        a = _i32(context)
        cap = max(int(d), 1)
        out = np.zeros(cap, np.int32)
        n, src, order = C.c_int(), C.c_int(), C.c_int()
        check(lib().dbl_store_lookup(self._h, _p32(a), len(a), int(d), _p32(out), cap,
                                     C.byref(n), C.byref(src), C.byref(order)))
        return LookupResult(out[:n.value].tolist(), SOURCES[src.value], order.value)

    def lookup_batch(self, contexts, depths):
        """Many independent lookups in one kernel launch (one CTA per query)."""
        ctxs = [_i32(c) for c in contexts]
        for c in ctxs:
            if len(c) == 0:
                raise InvalidArgument("lookup: empty context")
        offs = np.zeros(len(ctxs) + 1, np.int64)
        offs[1:] = np.cumsum([len(c) for c in ctxs])
        toks = np.concatenate(ctxs) if ctxs else np.zeros(1, np.int32)
        deps = _i32(depths)
        dcap = max(int(deps.max()) if len(deps) else 1, 1)
        nq = len(ctxs)
        oc = np.zeros(nq * dcap, np.int32)
        on, osrc, oord = (np.zeros(nq, np.int32) for _ in range(3))
        check(lib().dbl_store_lookup_batch(self._h, nq, offs.ctypes.data_as(C.POINTER(C.c_int64)),
                                           _p32(toks), _p32(deps), dcap, _p32(oc), _p32(on),
                                           _p32(osrc), _p32(oord)))
        return [LookupResult(oc[q * dcap:q * dcap + on[q]].tolist(), SOURCES[osrc[q]], int(oord[q]))
                for q in range(nq)]

    def record_accepted(self, tokens):  # datastore.cpp:134-137
        a = _i32(tokens)
        check(lib().dbl_store_record(self._h, DYNAMIC, _p32(a), len(a)))

    def record_rejected(self, tokens):  # datastore.cpp:139-142
        a = _i32(tokens)
        check(lib().dbl_store_record(self._h, REJECTED, _p32(a), len(a)))

    def flush_session(self):  # datastore.cpp:144-147
        check(lib().dbl_store_flush_session(self._h))

    def profile_lookup(self, context, d: int, iters: int = 100) -> float:
        """Device microseconds per lookup (back-to-back single-CTA lookups, CUDA events)."""
        ctx = _i32(context)
        v = C.c_double()
        check(lib().dbl_store_profile_lookup(self._h, _p32(ctx), len(ctx), int(d), int(iters), C.byref(v)))
        return v.value

    @property
    def stats(self) -> LookupStats:
        v = np.zeros(6, np.int64)
        check(lib().dbl_store_stats(self._h, v.ctypes.data_as(C.POINTER(C.c_int64))))
        return LookupStats(*[int(x) for x in v])


@dataclass
class NGramIndex:
    """A host-side NGramIndex value (datastore.hpp:19-27): the sequences and their steps.  Assign it to a
    store layer (``store.prior = idx``) to load it into HBM; the device layers answer lookups."""
    max_order: int = 3
    sequences: list = field(default_factory=list)
    steps: list = field(default_factory=list)

    def insert(self, tokens, step: int):  # datastore.cpp:9-12
        t = [int(x) for x in tokens]
        if not t:
            raise InvalidArgument("insert: empty token sequence")
        self.sequences.append(t)
        self.steps.append(int(step))

    def occurrence_count(self) -> int:  # datastore.cpp:22-26
        return sum(max(len(q) - k + 1, 0) for q in self.sequences for k in range(1, self.max_order + 1))

    def clear(self):
        self.sequences.clear()
        self.steps.clear()


def _flatten(seqs):
    off = np.zeros(len(seqs) + 1, np.int64)
    for i, q in enumerate(seqs):
        off[i + 1] = off[i] + len(q)
    flat = np.ascontiguousarray(np.concatenate([_i32(q) for q in seqs]) if seqs else np.zeros(1, np.int32))
    return flat, off


def build_prior(*args):
    """build_prior (datastore.cpp:149-159): the first K corpus sequences with step = index.

    ``build_prior(corpora, max_order, rounds) -> NGramIndex`` is the reference's signature (assign the
    result to ``store.prior``); ``build_prior(store, corpora, rounds)`` loads straight into
    ``store.prior`` (one bulk upload, dbl_build_prior) and returns the store."""
    if len(args) == 3 and isinstance(args[0], HierarchicalDatastore):
        store, corpora, rounds = args
        if rounds < 0:
            raise InvalidArgument("build_prior: rounds must be >= 0")
        seqs = [list(q) for q in list(corpora)[:rounds]]
        flat, off = _flatten(seqs)
        check(lib().dbl_build_prior(store._h, _i64(off), _p32(flat), len(seqs), int(store._orders[PRIOR]),
                                    len(seqs)))
        return store
    corpora, max_order, rounds = args
    if rounds < 0:
        raise InvalidArgument("build_prior: rounds must be >= 0")
    idx = NGramIndex(int(max_order))
    for i, q in enumerate(list(corpora)[:rounds]):
        idx.insert(q, i)
    return idx


def save_model(model: "TableModel", path: str):
    """save_model (model.cpp:230-234)"""
    with open(path, "w") as f:
        f.write(model.to_model_v1())


def load_model(path: str, device: int = 0) -> "TableModel":
    """load_model (model.cpp:236-242): model-v1 file -> device TableModel"""
    with open(path) as f:
        return TableModel.from_model_v1(f.read(), device)


def parse_dstore_v1(text: str):
    """dstore-v1 (datastore.cpp:161-187) -> (max_order, [sequences])."""
    lines = text.split("\n")
    if lines and lines[-1] == "":  # getline semantics: a trailing newline ends the last line
        lines.pop()
    head = lines[0].split() if lines else []
    if len(head) < 3 or head[0] != "dstore-v1":
        raise DoubleError("dstore-v1: bad header")
    n = int(head[2])
    if len(lines) - 1 < n:
        raise DoubleError("dstore-v1: truncated")
    return int(head[1]), [[int(t) for t in lines[1 + i].split()] for i in range(n)]


def serialize_index(max_order: int, sequences) -> str:
    """serialize_index (datastore.cpp:161-169): dstore-v1 text of one layer's sequences."""
    out = [f"dstore-v1 {int(max_order)} {len(sequences)}\n"]
    for seq in sequences:
        out.append(" ".join(str(int(t)) for t in seq) + "\n")
    return "".join(out)


def save_index(layer_or_store, path: str):
    """save_index (datastore.cpp:189-193) of a device layer (a HierarchicalDatastore saves its prior)."""
    layer = layer_or_store.prior if isinstance(layer_or_store, HierarchicalDatastore) else layer_or_store
    with open(path, "w") as f:
        f.write(serialize_index(layer.max_order, layer.sequences))


def load_index(path: str, store: "HierarchicalDatastore | None" = None, layer: int = PRIOR):
    """load_index (datastore.cpp:195-201) -> (max_order, sequences); with `store`, the sequences are
    inserted into that layer with step = index, as parse_index does (datastore.cpp:171-187)."""
    with open(path) as f:
        mo, seqs = parse_dstore_v1(f.read())
    if store is not None:
        lay = (store.prior, store.dynamic, store.rejected)[layer]
        lay.max_order = mo
        for i, sq in enumerate(seqs):
            lay.insert(sq, i)
    return mo, seqs


def _g17(x: float) -> str:  # std::snprintf("%.17g") (model.cpp:155-161, 176)
    return "%.17g" % float(x)


def serialize_model(order: int, vocab: int, windows, probs, fallback, smoothing: float = 0.1) -> str:
    """serialize_model (model.cpp:174-190): model-v1 text; rows in std::map (lexicographic window) order."""
    w = np.asarray(windows, np.int64).reshape(-1, order) if order else np.zeros((0, 0), np.int64)
    pr = np.asarray(probs, np.float64).reshape(-1, vocab)
    out = [f"model-v1 {int(vocab)} {int(order)} {_g17(smoothing)}\n"]
    for i in sorted(range(len(w)), key=lambda r: tuple(w[r])):
        out.append(" ".join(str(int(t)) for t in w[i]) + " :" + "".join(" " + _g17(v) for v in pr[i]) + "\n")
    out.append("fallback :" + "".join(" " + _g17(v) for v in np.asarray(fallback, np.float64)) + "\n")
    return "".join(out)


def parse_model_v1_smoothing(text: str) -> float:
    """the smoothing field of a model-v1 header (model.cpp:199-205)"""
    head = text.split("\n", 1)[0].split()
    if len(head) < 4 or head[0] != "model-v1":
        raise DoubleError("model-v1: bad header")
    return float(head[3])


def parse_model_v1(text: str):
    """model-v1 (model.cpp:199-228) -> (order, vocab, windows[n,order], probs[n,vocab], fallback)."""
    lines = text.split("\n")
    head = lines[0].split()
    if len(head) < 4 or head[0] != "model-v1":
        raise DoubleError("model-v1: bad header")
    vocab, order = int(head[1]), int(head[2])
    windows, rows, fallback = [], [], None
    for ln in lines[1:]:
        if not ln.strip():
            continue
        left, right = ln.split(":", 1)
        probs = np.array(right.split(), dtype=np.float64)
        if len(probs) != vocab:
            raise DoubleError("model-v1: truncated probability row")
        if left.strip() == "fallback":
            fallback = probs
            continue
        w = [int(t) for t in left.split()]
        if len(w) != order:
            raise DoubleError("model-v1: window length mismatch")
        windows.append(w)
        rows.append(probs)
    if fallback is None:
        raise DoubleError("model-v1: missing fallback row")
    return (order, vocab, np.array(windows, np.int32).reshape(-1, order),
            np.array(rows, np.float64).reshape(-1, vocab), fallback)


class _Model:
    _h = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().dbl_model_destroy(h)
            self._h = None

    @property
    def vocab_size(self) -> int:
        v = C.c_int()
        check(lib().dbl_model_vocab(self._h, C.byref(v)))
        return v.value

    @property
    def weight_bytes(self) -> int:
        v = C.c_int64()
        check(lib().dbl_model_weight_bytes(self._h, C.byref(v)))
        return v.value


class TableModel(_Model):
    """Device TableModel (model.hpp:18-25): order-m windows -> fp64 next-token rows."""

    def __init__(self, order, vocab, windows, probs, fallback, device: int = 0):
        w = np.ascontiguousarray(windows, np.int32).reshape(-1)
        p = np.ascontiguousarray(probs, np.float64).reshape(-1)
        f = np.ascontiguousarray(fallback, np.float64)
        n_rows = len(w) // order if order else 0
        h = C.c_void_p()
        check(lib().dbl_table_create(int(order), int(vocab), n_rows, _p32(w),
                                     p.ctypes.data_as(C.POINTER(C.c_double)),
                                     f.ctypes.data_as(C.POINTER(C.c_double)), int(device), C.byref(h)))
        self._h = h
        self.order = order
        # host image for serialize_model / save_model (the device copy is the one the loop reads)
        self._host = (int(order), int(vocab), w.reshape(-1, order) if order else w, p.reshape(-1, vocab), f)
        self.smoothing = 0.1

    @classmethod
    def from_model_v1(cls, text: str, device: int = 0) -> "TableModel":
        order, vocab, w, p, f = parse_model_v1(text)
        m = cls(order, vocab, w, p, f, device)
        m.smoothing = parse_model_v1_smoothing(text)
        return m

    def to_model_v1(self) -> str:
        """serialize_model (model.cpp:174-190)"""
        order, vocab, w, p, f = self._host
        return serialize_model(order, vocab, w, p, f, self.smoothing)


class Transformer(_Model):
    """Random-init bf16 transformer on the device (shapes: models.py presets)."""

    def __init__(self, cfg: TransformerConfig, device: int = 0, nccl_comm: int | None = None):
        h = C.c_void_p()
        check(lib().dbl_transformer_create(C.byref(cfg), int(device),
                                           C.c_void_p(nccl_comm) if nccl_comm else None, C.byref(h)))
        self._h = h
        self.cfg = cfg

    def weight(self, name: str, layer: int = -1, shape=None) -> np.ndarray:
        """bf16 weight -> np.float32 (for the torch fp32 reference in tests)."""
        numel = int(np.prod(shape))
        out = np.zeros(numel, np.uint16)
        check(lib().dbl_transformer_get_weight(self._h, name.encode(), int(layer),
                                               out.ctypes.data_as(C.POINTER(C.c_uint16)), numel))
        return (out.astype(np.uint32) << 16).view(np.float32).reshape(shape)


class TpTransformer(_Model):
    """Tensor-parallel target: len(devices) shards of `cfg` (column-parallel QKV /
    gate|up, row-parallel O / down, vocab-parallel LM head) exchanging partial sums inside the forward
    kernel.  Devices may repeat (shards co-reside on one GPU) or be distinct GPUs over NVLink."""

    def __init__(self, cfg: TransformerConfig, devices=(0, 0)):
        h = C.c_void_p()
        dv = _i32(devices)
        check(lib().dbl_tp_transformer_create(C.byref(cfg), _p32(dv), len(dv), C.byref(h)))
        self._h = h
        self.cfg = cfg
        self.devices = list(devices)


def forward_batch(model: _Model, context, candidates) -> list:
    """forward_batch (model.cpp:37-53) consumed greedily: argmax of each of the |cands|+1 rows."""
    ctx, cands = _i32(context), _i32(candidates)
    out = np.zeros(len(cands) + 1, np.int32)
    check(lib().dbl_forward_argmax(model._h, _p32(ctx), len(ctx), _p32(cands), len(cands), _p32(out)))
    return out.tolist()


def forward_logits(model: _Model, context, candidates) -> np.ndarray:
    """(|cands|+1) x vocab fp32 logits (tables: the fp64 probabilities rounded to fp32)."""
    ctx, cands = _i32(context), _i32(candidates)
    out = np.zeros((len(cands) + 1, model.vocab_size), np.float32)
    check(lib().dbl_forward_logits(model._h, _p32(ctx), len(ctx), _p32(cands), len(cands),
                                   out.ctypes.data_as(C.POINTER(C.c_float))))
    return out


def forward_dists(model: _Model, context, candidates) -> np.ndarray:
    """forward_batch's ProbVector rows (model.cpp:37-53), (|cands|+1) x vocab fp64: the rows the
    sampled decode loop consumes (tables exact; transformers softmax of the logits)."""
    ctx, cands = _i32(context), _i32(candidates)
    out = np.zeros((len(cands) + 1, model.vocab_size), np.float64)
    check(lib().dbl_forward_dists(model._h, _p32(ctx), len(ctx), _p32(cands), len(cands),
                                  out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


@dataclass
class PipelineOptions:  # pipeline.hpp:36-44 (+ LatencyConfig, :15-29)
    gamma: int = 4
    depth: int = 10
    draft_retrieval: bool = True
    target_retrieval: bool = True
    engine: str = "serial"  # serial|concurrent: identical results; the device always overlaps
    t_target: float = 1.0
    t_draft: float = 0.25
    t_lookup: float = 0.0
    t_sync: float = 0.0
    use_graphs: bool = True
    temperature: float = 0.0  # SamplerConfig (model.hpp:11-14): 0 = greedy
    rng_seed: int = 0

    def _c(self) -> _Opts:
        return _Opts(self.gamma, self.depth, int(self.draft_retrieval), int(self.target_retrieval),
                     int(self.engine == "concurrent"), self.t_target, self.t_draft, self.t_lookup,
                     self.t_sync, int(self.use_graphs), float(self.temperature), int(self.rng_seed))


@dataclass
class RunResult:  # pipeline.hpp:84-88
    output: list
    metrics: dict
    jsonl: str = ""
    traces: list = field(default_factory=list)


def _finish(rc, out, n, m, js, jl, want_jsonl) -> RunResult:
    import json
    if rc != 0 and want_jsonl and lib().dbl_last_error().decode().startswith("jsonl buffer too small"):
        # tokens and metrics were written; the traces outgrew the guess: fetch them at their size
        js = C.create_string_buffer(int(jl.value) + 1)
        rc = lib().dbl_last_run_jsonl(js, len(js), C.byref(jl))
    check(rc)
    text = js.value.decode() if want_jsonl else ""
    return RunResult(out[:n.value].tolist(), m.as_dict(), text,
                     [json.loads(x) for x in text.splitlines()] if want_jsonl else [])


def _jsonl_buf(max_new, gamma=1):
    return C.create_string_buffer(max(1 << 16, 512 * (max_new + 8)))


def run(draft: _Model, target: _Model, store: HierarchicalDatastore, prompt, max_new_tokens: int,
        opts: PipelineOptions | None = None, want_jsonl: bool = True) -> RunResult:
    """run (pipeline.cpp:264-323): the DOUBLE loop on the device."""
    opts = opts or PipelineOptions()
    p = _i32(prompt)
    cap = max(int(max_new_tokens), 1)
    out = np.zeros(cap, np.int32)
    n = C.c_int()
    m = RunMetrics()
    js = _jsonl_buf(max_new_tokens) if want_jsonl else None
    jl = C.c_int64()
    o = opts._c()
    rc = lib().dbl_run(draft._h, target._h, store._h, _p32(p), len(p), int(max_new_tokens),
                       C.byref(o), _p32(out), cap, C.byref(n), C.byref(m), js,
                       len(js) if js is not None else 0, C.byref(jl))
    return _finish(rc, out, n, m, js, jl, want_jsonl)


def last_run_log() -> np.ndarray:
    """Decision log of this thread's last run() (include/double_b200.h: dbl_last_run_log)."""
    n = C.c_int64()
    check(lib().dbl_last_run_log(None, 0, C.byref(n)))
    buf = np.zeros(max(n.value, 1), np.int32)
    check(lib().dbl_last_run_log(_p32(buf), len(buf), C.byref(n)))
    return buf[:n.value]


def set_exact_sampling(on: bool = True):
    """Sampled decoding at wide vocabularies on the reference-exact path (sequential fp64 sums and
    scan, fp64 pow — include/double_b200.h: dbl_set_exact_sampling); every visible device."""
    check(lib().dbl_set_exact_sampling(1 if on else 0))


def run_vanilla_ar(target: _Model, prompt, max_new_tokens: int, t_target: float = 1.0,
                   want_jsonl: bool = True, temperature: float = 0.0, rng_seed: int = 0) -> RunResult:
    """run_vanilla_ar (harness.cpp:233-258); temperature > 0 samples with the reference's AR stream."""
    p = _i32(prompt)
    cap = max(int(max_new_tokens), 1)
    out = np.zeros(cap, np.int32)
    n = C.c_int()
    m = RunMetrics()
    js = _jsonl_buf(max_new_tokens) if want_jsonl else None
    jl = C.c_int64()
    rc = lib().dbl_run_ar_sampled(target._h, _p32(p), len(p), int(max_new_tokens), float(t_target),
                                  float(temperature), C.c_uint64(int(rng_seed)), _p32(out), cap, C.byref(n),
                                  C.byref(m), js, len(js) if js is not None else 0, C.byref(jl))
    return _finish(rc, out, n, m, js, jl, want_jsonl)


def link_tp_processes(shard: "Transformer", group=None):
    """One process per GPU: link this process's tensor-parallel shard (tp_rank = this
    rank of `group`) with the other ranks' shards — CUDA IPC handles of the exchange buffers,
    all-gathered with torch.distributed (any backend; gloo is enough).  Afterwards every rank runs the
    same decode loop; the forwards exchange partial tiles inside fwd_kernel."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if shard.cfg.tp_size != world or shard.cfg.tp_rank != dist.get_rank(group):
        raise InvalidArgument("link_tp_processes: the shard's tp_rank / tp_size must be this rank / world size")
    buf = (C.c_uint8 * 256)()
    check(lib().dbl_tp_ipc_export(shard._h, buf, 256))
    flat = gather_tp_handles(bytes(buf), group)
    check(lib().dbl_tp_ipc_import(shard._h, flat, world))


def gather_tp_handles(mine: bytes, group=None) -> bytes:
    """Every rank's exchange-buffer handles (256 bytes each), concatenated in rank order."""
    import torch.distributed as dist
    if len(mine) != 256:
        raise InvalidArgument("gather_tp_handles: 4 CUDA IPC handles (256 bytes) per rank")
    allh = [None] * dist.get_world_size(group)
    dist.all_gather_object(allh, mine, group=group)
    return b"".join(allh)


def run_batch(draft: _Model, target: _Model, stores, prompts, max_new_tokens: int,
              opts: PipelineOptions | None = None, want_jsonl: bool = True):
    """Batched DOUBLE: run() for several independent sequences — one datastore each —
    sharing every draft-segment and verify forward.  Returns one RunResult per sequence, each equal to
    that sequence's own run()."""
    import json
    opts = opts or PipelineOptions()
    ps = [_i32(p) for p in prompts]
    B = len(ps)
    off = np.zeros(B + 1, np.int64)
    off[1:] = np.cumsum([len(p) for p in ps])
    toks = np.concatenate(ps) if ps else np.zeros(1, np.int32)
    n = max(int(max_new_tokens), 1)
    out = np.zeros(B * n, np.int32)
    out_n = np.zeros(max(B, 1), np.int32)
    mets = (RunMetrics * max(B, 1))()
    hs = (C.c_void_p * max(B, 1))(*[s._h.value if isinstance(s._h, C.c_void_p) else s._h for s in stores])
    js = C.create_string_buffer(B * max(1 << 16, 512 * (n + 8))) if want_jsonl else None
    jl = np.zeros(max(B, 1), np.int64)
    o = opts._c()
    check(lib().dbl_run_batch(draft._h, target._h, B, hs, off.ctypes.data_as(C.POINTER(C.c_int64)), _p32(toks),
                              int(max_new_tokens), C.byref(o), _p32(out), _p32(out_n), mets, js,
                              len(js) if js is not None else 0, jl.ctypes.data_as(C.POINTER(C.c_int64))))
    res, at = [], 0
    raw = js.raw if want_jsonl else b""
    for b in range(B):
        text = raw[at:at + jl[b]].decode() if want_jsonl else ""
        at += int(jl[b])
        res.append(RunResult(out[b * n: b * n + out_n[b]].tolist(), mets[b].as_dict(), text,
                             [json.loads(x) for x in text.splitlines()] if want_jsonl else []))
    return res


def run_vanilla_ar_batch(target: _Model, prompts, max_new_tokens: int):
    """Batched serving: run_vanilla_ar for several prompts in lockstep, one forward per step over all of
    them.  Returns (outputs, {"device_ms", "tokens", "kernel_launches"})."""
    ps = [_i32(p) for p in prompts]
    off = np.zeros(len(ps) + 1, np.int64)
    off[1:] = np.cumsum([len(p) for p in ps])
    toks = np.concatenate(ps) if ps else np.zeros(1, np.int32)
    n = max(int(max_new_tokens), 1)
    out = np.zeros(len(ps) * n, np.int32)
    out_n = np.zeros(max(len(ps), 1), np.int32)
    ms, launches = C.c_double(), C.c_int64()
    check(lib().dbl_run_ar_batch(target._h, len(ps), off.ctypes.data_as(C.POINTER(C.c_int64)), _p32(toks),
                                 int(max_new_tokens), _p32(out), _p32(out_n), C.byref(ms), C.byref(launches)))
    outs = [out[b * int(max_new_tokens): b * int(max_new_tokens) + out_n[b]].tolist() for b in range(len(ps))]
    return outs, {"device_ms": ms.value, "tokens": int(sum(out_n[:len(ps)])), "kernel_launches": launches.value}


def run_serial_sd(draft: _Model, target: _Model, store: HierarchicalDatastore, prompt,
                  max_new_tokens: int, opts: PipelineOptions | None = None,
                  use_retrieval: bool = False, want_jsonl: bool = True) -> RunResult:
    """run_serial_sd (harness.cpp:264-369): methods ``sd`` / ``draft_retrieval``."""
    opts = opts or PipelineOptions()
    p = _i32(prompt)
    cap = max(int(max_new_tokens), 1)
    out = np.zeros(cap, np.int32)
    n = C.c_int()
    m = RunMetrics()
    js = _jsonl_buf(max_new_tokens) if want_jsonl else None
    jl = C.c_int64()
    o = opts._c()
    rc = lib().dbl_run_serial_sd(draft._h, target._h, store._h, _p32(p), len(p),
                                 int(max_new_tokens), C.byref(o), int(use_retrieval), _p32(out), cap,
                                 C.byref(n), C.byref(m), js, len(js) if js is not None else 0,
                                 C.byref(jl))
    return _finish(rc, out, n, m, js, jl, want_jsonl)


# ------------------------------------------------------------------------------ verifier + RNG
# specpar::Rng / derive_rng (rng.hpp:19-35) and the verifier interface (verification.hpp:30-53),
# computed on the device (verify.cu) with the reference's draw order and fp64 summation order.
class Rng:  # rng.hpp:19-30 — the mt19937_64 stream lives on the device
    def __init__(self, seed: int = 0, device: int = 0, _handle=None):
        if _handle is None:
            h = C.c_void_p()
            check(lib().dbl_rng_create(C.c_uint64(seed), device, C.byref(h)))
            _handle = h
        self._h = _handle

    def uniform(self, n: int | None = None):
        k = 1 if n is None else n
        out = np.zeros(max(k, 1), np.float64)
        check(lib().dbl_rng_uniform(self._h, out.ctypes.data_as(C.POINTER(C.c_double)), k))
        return float(out[0]) if n is None else out[:k]

    def __del__(self):
        try:
            if self._h:
                lib().dbl_rng_destroy(self._h)
        except Exception:  # noqa: BLE001 (interpreter shutdown)
            pass


def derive_rng(seed: int, round_: int, lane: int, device: int = 0) -> Rng:  # rng.hpp:33-35
    h = C.c_void_p()
    check(lib().dbl_rng_derive(C.c_uint64(seed), C.c_uint64(round_), C.c_uint64(lane), device, C.byref(h)))
    return Rng(_handle=h)


def _rows(rows):
    """ragged fp64 rows (list of ProbVector) -> (flat, offsets, n)"""
    rows = [np.asarray(r, np.float64).reshape(-1) for r in (rows or [])]
    off = np.zeros(len(rows) + 1, np.int64)
    for i, r in enumerate(rows):
        off[i + 1] = off[i] + len(r)
    flat = np.ascontiguousarray(np.concatenate(rows) if rows else np.zeros(1), np.float64)
    return flat, off, len(rows)


def _f64(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _i64(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


VERIFY_KINDS = ["all_accepted", "correction", "extension", "residual_correction"]  # to_string(VerifyKind)


@dataclass
class GuidanceChain:  # verification.hpp:13-17
    tokens: list = field(default_factory=list)
    probs: list = field(default_factory=list)
    matched_len: int = 0


@dataclass
class VerifyOutcome:  # verification.hpp:22-26
    accepted_len: int
    committed: list
    kind: str


def accept_prob(p, q, x: int) -> float:  # verification.cpp:19-23
    p = np.ascontiguousarray(p, np.float64)
    q = np.ascontiguousarray(q, np.float64)
    out = C.c_double()
    check(lib().dbl_accept_prob(_f64(p), len(p), _f64(q), len(q), x, C.byref(out)))
    return out.value


def residual_sample(p, q, rng: Rng) -> int:  # verification.cpp:40-50
    p = np.ascontiguousarray(p, np.float64)
    q = np.ascontiguousarray(q, np.float64)
    out = C.c_int32()
    check(lib().dbl_residual_sample(_f64(p), len(p), _f64(q), len(q), rng._h, C.byref(out)))
    return out.value


def residual_sample_point_mass(p, x: int, rng: Rng) -> int:  # verification.cpp:52-58
    p = np.ascontiguousarray(p, np.float64)
    out = C.c_int32()
    check(lib().dbl_residual_sample_point_mass(_f64(p), len(p), x, rng._h, C.byref(out)))
    return out.value


def verify_against_target(draft_tokens, draft_probs, target_probs, temperature: float, rng: Rng):
    """verification.cpp:60-78: the first rejected index, or None (std::nullopt)"""
    d = _i32(draft_tokens)
    dp, doff, nd = _rows(draft_probs)
    tp, toff, nt = _rows(target_probs)
    out = C.c_int()
    check(lib().dbl_verify_against_target(_p32(d), len(d), _f64(dp), _i64(doff), nd, _f64(tp), _i64(toff), nt,
                                          float(temperature), rng._h, C.byref(out)))
    return None if out.value < 0 else out.value


def guided_output(draft_tokens, draft_probs, guidance: GuidanceChain, first_reject, temperature: float,
                  rng: Rng) -> VerifyOutcome:  # verification.cpp:80-132
    d = _i32(draft_tokens)
    dp, doff, nd = _rows(draft_probs)
    gt = _i32(guidance.tokens)
    gp, goff, ng = _rows(guidance.probs)
    cap = len(d) + len(gt) + 1
    out = np.zeros(cap, np.int32)
    n, acc, kind = C.c_int(), C.c_int(), C.c_int()
    check(lib().dbl_guided_output(_p32(d), len(d), _f64(dp), _i64(doff), nd, _p32(gt), len(gt), _f64(gp),
                                  _i64(goff), ng, -1 if first_reject is None else int(first_reject),
                                  float(temperature), rng._h, _p32(out), cap, C.byref(n), C.byref(acc),
                                  C.byref(kind)))
    return VerifyOutcome(acc.value, out[:n.value].tolist(), VERIFY_KINDS[kind.value])


__all__ += ["Rng", "derive_rng", "GuidanceChain", "VerifyOutcome", "accept_prob", "residual_sample",
            "residual_sample_point_mass", "verify_against_target", "guided_output", "VERIFY_KINDS"]


# ------------------------------------------------------------------ model-level helpers (model.hpp:40-48)
def tempered(dist, temperature: float, device: int = 0) -> np.ndarray:  # model.cpp:55-68
    d = np.ascontiguousarray(dist, np.float64)
    out = np.zeros(max(len(d), 1), np.float64)
    check(lib().dbl_tempered(_f64(d), len(d), float(temperature), device, _f64(out)))
    return out[:len(d)]


def argmax_token(dist, device: int = 0) -> int:  # model.cpp:70-81
    d = np.ascontiguousarray(dist, np.float64)
    out = C.c_int32()
    check(lib().dbl_argmax_token(_f64(d) if len(d) else None, len(d), device, C.byref(out)))
    return out.value


def argmax_rows(rows, device: int = 0) -> list:
    """argmax_token of every row in one launch (one CTA per row, warp-shuffle reduction)."""
    flat, off, n = _rows(rows)
    out = np.zeros(max(n, 1), np.int32)
    check(lib().dbl_argmax_rows(_f64(flat), _i64(off), n, device, _p32(out)))
    return out[:n].tolist()


def sample(dist, temperature: float, rng: "Rng | None", device: int = 0) -> int:  # model.cpp:83-97
    d = np.ascontiguousarray(dist, np.float64)
    out = C.c_int32()
    check(lib().dbl_sample(_f64(d), len(d), float(temperature), rng._h if rng is not None else None, device,
                           C.byref(out)))
    return out.value


# ------------------------------------------------------------------ drafter (speculation.hpp:34-59)
@dataclass
class RetrievalResult:  # speculation.hpp:12-17
    emitted: list
    matched_len: int
    probs: list
    source: str = "miss"


@dataclass
class DraftChain:  # speculation.hpp:19-24
    segments: list
    tokens: list
    probs: list
    total_len: int


def _split_rows(flat: np.ndarray, lengths) -> list:
    out, at = [], 0
    for n in lengths:
        out.append(flat[at:at + n])
        at += n
    return out


def accept_with_model(dists, cands, temperature: float = 0.0, rng: "Rng | None" = None,
                      device: int = 0) -> RetrievalResult:  # speculation.cpp:7-52
    flat, off, n = _rows(dists)
    c = _i32(cands)
    em = np.zeros(len(c) + 1, np.int32)
    probs = np.zeros(max(int(off[-1]), 1), np.float64)
    res = _RetrievalC()
    check(lib().dbl_accept_with_model(_f64(flat), _i64(off), n, _p32(c), len(c), float(temperature),
                                      rng._h if rng is not None else None, device, _p32(em), len(em),
                                      _f64(probs), len(probs), C.byref(res)))
    lens = [int(off[i + 1] - off[i]) for i in range(res.n_probs)]
    return RetrievalResult(em[:res.n_emitted].tolist(), res.matched_len, _split_rows(probs, lens))


def retrieval_forward(model: "_Model", store: "HierarchicalDatastore | None", context, depth: int,
                      temperature: float = 0.0, rng: "Rng | None" = None, use_retrieval: bool = True,
                      want_probs: bool = True) -> RetrievalResult:  # speculation.cpp:54-66
    ctx = _i32(context)
    V = model.vocab_size
    em = np.zeros(max(int(depth), 0) + 1, np.int32)
    probs = np.zeros((int(depth) + 1) * V if want_probs else 1, np.float64)
    res = _RetrievalC()
    check(lib().dbl_retrieval_forward(model._h, store._h if store is not None else None, _p32(ctx), len(ctx),
                                      int(depth), float(temperature), rng._h if rng is not None else None,
                                      int(bool(use_retrieval)), _p32(em), len(em),
                                      _f64(probs) if want_probs else None, len(probs), C.byref(res)))
    return RetrievalResult(em[:res.n_emitted].tolist(), res.matched_len,
                           _split_rows(probs, [V] * res.n_probs) if want_probs else [], SOURCES[res.source])


def iterative_draft(model: "_Model", store: "HierarchicalDatastore | None", context, gamma: int, depth: int,
                    temperature: float = 0.0, rng: "Rng | None" = None, use_retrieval: bool = True,
                    want_probs: bool = True) -> DraftChain:  # speculation.cpp:68-86
    ctx = _i32(context)
    V = model.vocab_size
    cap = max(int(gamma), 1) * (max(int(depth), 0) + 1)
    toks = np.zeros(cap, np.int32)
    probs = np.zeros(cap * V if want_probs else 1, np.float64)
    segs = (_RetrievalC * max(int(gamma), 1))()
    n = C.c_int()
    check(lib().dbl_iterative_draft(model._h, store._h if store is not None else None, _p32(ctx), len(ctx),
                                    int(gamma), int(depth), float(temperature), rng._h if rng is not None else None,
                                    int(bool(use_retrieval)), segs, _p32(toks), cap, C.byref(n),
                                    _f64(probs) if want_probs else None, len(probs)))
    tokens = toks[:n.value].tolist()
    rows = _split_rows(probs, [V] * n.value) if want_probs else []
    out, at = [], 0
    for j in range(int(gamma)):
        k = segs[j].n_emitted
        out.append(RetrievalResult(tokens[at:at + k], segs[j].matched_len, rows[at:at + k], SOURCES[segs[j].source]))
        at += k
    return DraftChain(out, tokens, rows, n.value)


def measure_amt(traces) -> float:  # speculation.cpp:88-94
    m = _i32([t.matched_len if isinstance(t, RetrievalResult) else int(t) for t in traces])
    out = C.c_double()
    check(lib().dbl_measure_amt(_p32(m) if len(m) else None, len(m), C.byref(out)))
    return out.value


# ------------------------------------------------------------------ decoder state machine (pipeline.hpp)
MODES = ["pre_verify", "post_verify", "ar", "serial"]
KINDS = ["pending_reject", "extend_keep_draft", "extend_draft_subsumed", "extend_drop_draft", "ar_step", "reject",
         "all_accepted"]


@dataclass
class PipelineState:  # pipeline.hpp:46-55
    committed: list = field(default_factory=list)
    speculative: list = field(default_factory=list)
    spec_probs: list = field(default_factory=list)  # rows; greedy rows are not materialised (None entries)
    mode: str = "pre_verify"
    prev_tokens: int = 0
    round: int = 0
    clock: float = 0.0
    last_committed_len: int = 0


def _trace_dict(t) -> dict:  # RoundTrace (pipeline.hpp:57-71), keys in traces_to_jsonl order
    return {"round": t.round, "mode": MODES[t.mode], "pending": t.pending, "draft_len": t.draft_len,
            "draft_matched": list(t.draft_matched[:t.n_draft_matched]), "target_matched": t.target_matched,
            "target_source": SOURCES[t.target_source], "accepted_pending": t.accepted_pending,
            "pending_reject": bool(t.pending_reject), "rejected": bool(t.rejected), "committed": t.committed_count,
            "kind": KINDS[t.kind], "clock_delta": t.clock_delta}


def _trace_c(d: dict):
    from ._capi import RoundTrace as _T
    t = _T()
    t.round = int(d.get("round", 0))
    t.mode = MODES.index(d.get("mode", "pre_verify"))
    t.pending = int(d.get("pending", 0))
    t.draft_len = int(d.get("draft_len", 0))
    dm = list(d.get("draft_matched", []))
    t.n_draft_matched = len(dm)
    for i, v in enumerate(dm):
        t.draft_matched[i] = int(v)
    t.target_matched = int(d.get("target_matched", -1))
    t.target_source = SOURCES.index(d.get("target_source", "miss"))
    t.accepted_pending = int(d.get("accepted_pending", 0))
    t.pending_reject = int(bool(d.get("pending_reject", False)))
    t.rejected = int(bool(d.get("rejected", False)))
    t.committed_count = int(d.get("committed", d.get("committed_count", 0)))
    t.kind = KINDS.index(d.get("kind", "extend_draft_subsumed"))
    t.clock_delta = float(d.get("clock_delta", 0.0))
    return t


def _traces_c(traces):
    from ._capi import RoundTrace as _T
    arr = (_T * max(len(traces), 1))()
    for i, d in enumerate(traces):
        arr[i] = _trace_c(d)
    return arr


def rollback(state: PipelineState, keep_len: int):  # pipeline.cpp:15-30 (through the C-ABI)
    st = _StateC()
    com = _i32(state.committed)
    st.committed, st.n_committed, st.committed_cap = _p32(com), len(com), len(com)
    st.n_speculative = st.speculative_cap = len(state.speculative)
    st.n_spec_probs = len(state.spec_probs)
    st.mode = MODES.index(state.mode)
    st.last_committed_len = int(state.last_committed_len)
    check(lib().dbl_rollback(C.byref(st), int(keep_len)))
    state.committed = com[:st.n_committed].tolist()
    state.speculative, state.spec_probs, state.mode = [], [], "pre_verify"


class Session:
    """The device lanes (token buffers + KV) one PipelineState runs on between rounds."""

    def __init__(self, draft: "_Model", target: "_Model"):
        h = C.c_void_p()
        check(lib().dbl_session_create(draft._h, target._h, C.byref(h)))
        self._h, self._models = h, (draft, target)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                lib().dbl_session_destroy(h)
            except Exception:  # noqa: BLE001 (interpreter shutdown)
                pass
            self._h = None


_SESSIONS: dict = {}


def run_round(state: PipelineState, draft: "_Model", target: "_Model", store: "HierarchicalDatastore",
              opts: "PipelineOptions | None" = None, session: Session | None = None) -> dict:
    """run_round (pipeline.cpp:223-262): one DOUBLE round on the device; `state` advances in place and the
    round's trace is returned.  Without an explicit session the (draft, target) pair's cached one is used."""
    opts = opts or PipelineOptions()
    if session is None:
        key = (id(draft), id(target))
        session = _SESSIONS.get(key)
        if session is None or session._models != (draft, target):
            session = _SESSIONS[key] = Session(draft, target)
    V = target.vocab_size
    gd = opts.gamma * (opts.depth + 1)
    ncom = len(state.committed) + len(state.speculative) + opts.depth + 1
    com = np.zeros(max(ncom, 1), np.int32)
    com[:len(state.committed)] = state.committed
    spec = np.zeros(max(gd, len(state.speculative), 1), np.int32)
    spec[:len(state.speculative)] = state.speculative
    st = _StateC()
    st.committed, st.n_committed, st.committed_cap = _p32(com), len(state.committed), len(com)
    st.speculative, st.n_speculative, st.speculative_cap = _p32(spec), len(state.speculative), len(spec)
    st.n_spec_probs = len(state.spec_probs)
    probs = None
    if opts.temperature != 0.0:
        rows = max(gd, len(state.speculative), 1)
        probs = np.zeros(rows * V, np.float64)
        have = [r for r in state.spec_probs if r is not None]
        if len(have) == len(state.speculative):
            if have:
                probs[:len(have) * V] = np.concatenate([np.asarray(r, np.float64) for r in have])
            st.spec_probs = _f64(probs)  # rows in, the new tail's rows out
        else:
            st.spec_probs = None  # the session's own device rows from its previous round
        st.spec_probs_cap = rows
    st.mode = MODES.index(state.mode)
    st.prev_tokens = int(state.prev_tokens)
    st.round = int(state.round)
    st.clock = float(state.clock)
    st.last_committed_len = int(state.last_committed_len)
    o = opts._c()
    tr = _TraceC()
    check(lib().dbl_run_round(session._h, store._h, C.byref(o), C.byref(st), C.byref(tr)))
    if not st.spec_probs:
        probs = None
    state.committed = com[:st.n_committed].tolist()
    state.speculative = spec[:st.n_speculative].tolist()
    if opts.temperature != 0.0 and probs is not None:
        state.spec_probs = [probs[i * V:(i + 1) * V].copy() for i in range(st.n_speculative)]
    else:
        state.spec_probs = [None] * st.n_speculative
    state.mode = MODES[st.mode]
    state.prev_tokens = st.prev_tokens
    state.round = st.round
    state.clock = st.clock
    state.last_committed_len = st.last_committed_len
    return _trace_dict(tr)


def compute_metrics(traces, t_target: float = 1.0) -> dict:  # pipeline.cpp:325-371
    m = RunMetrics()
    arr = _traces_c(traces)
    check(lib().dbl_compute_metrics(arr, len(traces), float(t_target), C.byref(m)))
    d = m.as_dict()
    return {k: d[k] for k in ("tokens", "rounds", "clock", "m", "amt", "speedup")}


def traces_to_jsonl(traces) -> str:  # pipeline.cpp:373-394
    arr = _traces_c(traces)
    n = C.c_int64()
    check(lib().dbl_traces_to_jsonl(arr, len(traces), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(lib().dbl_traces_to_jsonl(arr, len(traces), buf, len(buf), C.byref(n)))
    return buf.value.decode()


def write_traces(traces, path: str):  # pipeline.cpp:396-400
    check(lib().dbl_write_traces(_traces_c(traces), len(traces), str(path).encode()))


from ._capi import PipelineStateC as _StateC, RetrievalResult as _RetrievalC, RoundTrace as _TraceC  # noqa: E402

__all__ += ["tempered", "argmax_token", "argmax_rows", "sample", "RetrievalResult", "DraftChain",
            "accept_with_model", "retrieval_forward", "iterative_draft", "measure_amt", "PipelineState",
            "rollback", "Session", "run_round", "compute_metrics", "traces_to_jsonl", "write_traces", "MODES",
            "KINDS"]
