"""The reference's experiment harness in front of the device decode loop (the callers
and set-up either side of the path): key=value configs, the synthetic corpus, table models built from
it, the datastore prior and the six methods — so a reference config file (e.g.
proj/configs/ceiling_break.cfg) runs unchanged on the B200.

    parse_config / load_config / serialize_config   harness.cpp:37-149
    gen_corpus                                      harness.cpp:151-186
    build_model_from_corpus                         model.cpp:98-152
    build_setup / build_store                       harness.cpp:188-210
    run_method_on / run_method                      harness.cpp:403-433

Host-side set-up only: the corpus / model build is O(corpus) Python, every decode runs through the
device library (run, run_serial_sd, run_vanilla_ar)."""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from ._capi import DoubleError, InvalidArgument
from .specpar import (HierarchicalDatastore, PipelineOptions, TableModel, run, run_serial_sd,
                      run_vanilla_ar)

METHODS = ["vanilla_ar", "sd", "psd", "target_retrieval", "draft_retrieval", "double"]  # harness.cpp:11-20
BOS = 0  # kBosToken, types.hpp:15


# --------------------------------------------------------------------------------------- RNG
def splitmix64(x: int) -> int:  # rng.hpp:8-13
    x = (x + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    x = ((x ^ (x >> 27)) * 0x94D49BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return x ^ (x >> 31)


class _MT64:
    """std::mt19937_64 (the engine of specpar::Rng, rng.hpp:19-30) — host-side, for set-up only."""

    def __init__(self, seed: int):
        M = 0xFFFFFFFFFFFFFFFF
        self.mt = [seed & M]
        for i in range(1, 312):
            p = self.mt[-1]
            self.mt.append((6364136223846793005 * (p ^ (p >> 62)) + i) & M)
        self.idx = 312

    def next(self) -> int:
        if self.idx >= 312:
            mt = self.mt
            for i in range(312):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + 156) % 312] ^ xa
            self.idx = 0
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF

    def uniform(self) -> float:  # Rng::uniform, rng.hpp:23
        return (self.next() >> 11) * (1.0 / 9007199254740992.0)


# ------------------------------------------------------------------------------------ config
@dataclass
class ExperimentConfig:  # harness.hpp:21-43 (defaults as shipped)
    vocab: int = 32
    rho: float = 0.5
    corpus_len: int = 4096
    draft_order: int = 1
    target_order: int = 2
    smoothing: float = 0.1
    t_target: float = 1.0
    t_draft: float = 0.25
    t_lookup: float = 0.0
    t_sync: float = 0.0
    gamma: int = 0
    depth: int = 10
    ngram: int = 3
    prior_rounds: int = 10
    temperature: float = 0.0
    seed: int = 1
    method: str = "double"
    max_new_tokens: int = 256
    prompt_len: int = 8
    rejected_cache: bool = True
    engine: str = "serial"

    def effective_gamma(self) -> int:  # harness.cpp:32-35
        if self.gamma > 0:
            return self.gamma
        if self.t_draft <= 0.0:
            raise InvalidArgument("t_draft must be > 0")
        return int(math.ceil(self.t_target / self.t_draft))

    def validate(self):  # harness.cpp:37-53
        def bad(msg):
            raise InvalidArgument(msg)
        if self.vocab < 4:
            bad("vocab must be >= 4")
        if self.rho < 0.0 or self.rho > 1.0:
            bad("rho out of [0,1]")
        if self.corpus_len < self.prompt_len + 1:
            bad("corpus too short")
        if self.draft_order < 1 or self.target_order < 1:
            bad("model orders must be >= 1")
        if self.smoothing < 0.0:
            bad("smoothing must be >= 0")
        if self.t_target < 0.0 or self.t_draft <= 0.0 or self.t_lookup < 0.0 or self.t_sync < 0.0:
            bad("latency values out of range")
        if self.gamma < 0:
            bad("gamma must be >= 0")
        if self.depth < 1:
            bad("depth must be >= 1")
        if self.ngram < 1:
            bad("ngram must be >= 1")
        if self.prior_rounds < 0:
            bad("prior_rounds must be >= 0")
        if self.temperature < 0.0:
            bad("temperature must be >= 0")
        if self.max_new_tokens < 1:
            bad("max_new_tokens must be >= 1")
        if self.prompt_len < 1:
            bad("prompt_len must be >= 1")


_INT = {"vocab", "corpus_len", "draft_order", "target_order", "gamma", "depth", "ngram", "prior_rounds",
        "seed", "max_new_tokens", "prompt_len"}
_FLOAT = {"rho", "smoothing", "t_target", "t_draft", "t_lookup", "t_sync", "temperature"}


def parse_config(text: str) -> ExperimentConfig:
    """parse_config (harness.cpp:55-114): key=value lines, '#' comments; unknown keys and bad values
    are errors (runtime_error with the line number, as the reference)."""
    cfg = ExperimentConfig()
    for lineno, line in enumerate(text.split("\n"), 1):
        line = line.split("#", 1)[0]
        if "=" not in line:
            if line.strip(" \t\r"):
                raise DoubleError(f"config line {lineno}: expected key=value")
            continue
        key, val = (x.strip(" \t\r") for x in line.split("=", 1))
        try:
            if key in _INT:
                setattr(cfg, key, int(val, 10))
            elif key in _FLOAT:
                setattr(cfg, key, float(val))
            elif key == "method":
                if val not in METHODS:
                    raise ValueError
                cfg.method = val
            elif key == "rejected_cache":
                cfg.rejected_cache = val in ("1", "true")
            elif key == "engine":
                if val not in ("serial", "concurrent"):
                    raise ValueError
                cfg.engine = val
            else:
                raise ValueError
        except ValueError:  # the reference maps unknown keys and bad values to the same error
            raise DoubleError(f"config line {lineno}: bad value for {key}") from None
    cfg.validate()
    return cfg


def load_config(path: str) -> ExperimentConfig:  # harness.cpp:116-122
    with open(path) as f:
        return parse_config(f.read())


def serialize_config(cfg: ExperimentConfig) -> str:  # harness.cpp:124-149 (key order as shipped)
    def g(x):  # std::ostream default formatting of a double (6 significant digits, %g)
        return f"{x:g}"
    return "".join([
        f"vocab={cfg.vocab}\n", f"rho={g(cfg.rho)}\n", f"corpus_len={cfg.corpus_len}\n",
        f"draft_order={cfg.draft_order}\n", f"target_order={cfg.target_order}\n",
        f"smoothing={g(cfg.smoothing)}\n", f"t_target={g(cfg.t_target)}\n", f"t_draft={g(cfg.t_draft)}\n",
        f"t_lookup={g(cfg.t_lookup)}\n", f"t_sync={g(cfg.t_sync)}\n", f"gamma={cfg.gamma}\n",
        f"depth={cfg.depth}\n", f"ngram={cfg.ngram}\n", f"prior_rounds={cfg.prior_rounds}\n",
        f"temperature={g(cfg.temperature)}\n", f"seed={cfg.seed}\n", f"method={cfg.method}\n",
        f"max_new_tokens={cfg.max_new_tokens}\n", f"prompt_len={cfg.prompt_len}\n",
        f"rejected_cache={1 if cfg.rejected_cache else 0}\n", f"engine={cfg.engine}\n"])


# ------------------------------------------------------------------------------------- setup
def gen_corpus(vocab: int, rho: float, length: int, seed: int):
    """gen_corpus (harness.cpp:151-186): fresh random spans mixed with replays of earlier spans at
    rate rho, split into 64-token sequences; the same mt19937_64 draws as the reference."""
    if vocab < 4:
        raise InvalidArgument("vocab must be >= 4")
    if rho < 0.0 or rho > 1.0:
        raise InvalidArgument("rho out of [0,1]")
    if length < 1:
        raise InvalidArgument("length must be >= 1")
    rng = _MT64(splitmix64((seed ^ 0x636F727075730000) & 0xFFFFFFFFFFFFFFFF))
    lo, hi = 1, vocab - 2  # clear of BOS and EOS
    stream = []
    while len(stream) < length:
        replay = len(stream) >= 4 and rng.uniform() < rho
        if replay:
            span = 4 + int(rng.uniform() * 13.0)
            start = int(rng.uniform() * float(len(stream)))
            end = min(start + span, len(stream))
            stream.extend(stream[start:end])
        else:
            span = 1 + int(rng.uniform() * 4.0)
            for _ in range(span):
                stream.append(lo + int(rng.uniform() * (hi - lo + 1)))
    stream = stream[:length]
    return [stream[i:i + 64] for i in range(0, len(stream), 64)]


def _window(order: int, ctx) -> tuple:  # window_of, model.cpp:13-21
    take = min(len(ctx), order)
    return tuple([BOS] * (order - take) + list(ctx[len(ctx) - take:]))


@dataclass
class TableSpec:
    """A TableModel's host image (model.hpp:18-25): windows / rows in std::map order + fallback."""
    order: int
    vocab: int
    smoothing: float
    windows: np.ndarray
    probs: np.ndarray
    fallback: np.ndarray

    def device(self, device: int = 0) -> TableModel:
        m = TableModel(self.order, self.vocab, self.windows, self.probs, self.fallback, device)
        m.smoothing = self.smoothing
        return m


def build_model_from_corpus(corpus, order: int, smoothing: float, vocab: int) -> TableSpec:
    """build_model_from_corpus (model.cpp:98-152): (count + smoothing)-normalised next-token rows per
    BOS-padded window; unseen windows fall back to the smoothed unigram distribution."""
    if not corpus:
        raise InvalidArgument("empty corpus")
    if order < 1:
        raise InvalidArgument("order must be >= 1")
    if smoothing < 0.0:
        raise InvalidArgument("smoothing must be >= 0")
    counts = {}
    glob = np.zeros(vocab, np.float64)
    for seq in corpus:
        for i, tok in enumerate(seq):
            if tok < 0 or tok >= vocab:
                raise InvalidArgument("corpus token out of range")
            glob[tok] += 1.0
            if i + 1 < len(seq):
                lo = i + 1 - order if i + 1 >= order else 0
                w = _window(order, seq[lo:i + 1])
                row = counts.get(w)
                if row is None:
                    row = counts[w] = np.zeros(vocab, np.float64)
                row[seq[i + 1]] += 1.0
    keys = sorted(counts)
    probs = np.zeros((len(keys), vocab), np.float64)
    for r, w in enumerate(keys):
        p = counts[w] + smoothing
        s = 0.0
        for v in p:  # the reference's sequential sum
            s += float(v)
        if s <= 0.0:
            raise DoubleError("empty count row")
        probs[r] = p / s
    gsum = 0.0
    for c in glob:
        gsum += float(c)
    sm = max(smoothing, 1e-12)
    fallback = (glob + sm) / (gsum + sm * vocab)
    windows = np.array(keys, np.int32).reshape(-1, order)
    return TableSpec(order, vocab, smoothing, windows, probs, fallback)


@dataclass
class ExperimentSetup:  # harness.hpp (build_setup's result)
    corpus: list
    draft: TableSpec
    target: TableSpec
    prompt: list = field(default_factory=list)


def build_setup(cfg: ExperimentConfig) -> ExperimentSetup:  # harness.cpp:188-202
    cfg.validate()
    corpus = gen_corpus(cfg.vocab, cfg.rho, cfg.corpus_len, cfg.seed)
    d = build_model_from_corpus(corpus, cfg.draft_order, cfg.smoothing, cfg.vocab)
    t = build_model_from_corpus(corpus, cfg.target_order, cfg.smoothing, cfg.vocab)
    if len(corpus[0]) < cfg.prompt_len:
        raise InvalidArgument("prompt_len exceeds the first corpus sequence")
    return ExperimentSetup(corpus, d, t, corpus[0][:cfg.prompt_len])


def build_store(cfg: ExperimentConfig, corpus, device: int = 0) -> HierarchicalDatastore:  # harness.cpp:204-210
    st = HierarchicalDatastore(cfg.ngram, cfg.depth, device)
    for i, seq in enumerate(corpus[:cfg.prior_rounds]):  # build_prior, datastore.cpp:149-159
        st.prior.insert(seq, i)
    st.rejected_enabled = cfg.rejected_cache
    return st


# ----------------------------------------------------------------------------------- methods
def run_method_on(cfg: ExperimentConfig, setup: ExperimentSetup, method: str | None = None, device: int = 0):
    """run_method_on (harness.cpp:403-429) on the device: the method's decode with the reference's
    options; returns the RunResult (output, metrics, traces_to_jsonl text)."""
    method = method or cfg.method
    if method not in METHODS:
        raise InvalidArgument(f"unknown method: {method}")
    d, t = setup.draft.device(device), setup.target.device(device)
    opts = PipelineOptions(gamma=cfg.effective_gamma(), depth=cfg.depth, t_target=cfg.t_target,
                           t_draft=cfg.t_draft, t_lookup=cfg.t_lookup, t_sync=cfg.t_sync,
                           temperature=cfg.temperature, rng_seed=cfg.seed, engine=cfg.engine)
    if method == "vanilla_ar":
        return run_vanilla_ar(t, setup.prompt, cfg.max_new_tokens, t_target=cfg.t_target,
                              temperature=cfg.temperature, rng_seed=cfg.seed)
    st = build_store(cfg, setup.corpus, device)
    if method in ("sd", "draft_retrieval"):
        return run_serial_sd(d, t, st, setup.prompt, cfg.max_new_tokens, opts,
                             use_retrieval=method == "draft_retrieval")
    opts.draft_retrieval = method == "double"
    opts.target_retrieval = method in ("double", "target_retrieval")
    return run(d, t, st, setup.prompt, cfg.max_new_tokens, opts)


def run_method(cfg: ExperimentConfig, device: int = 0):  # harness.cpp:431-434
    return run_method_on(cfg, build_setup(cfg), cfg.method, device)


def run_config(text: str, method: str | None = None, device: int = 0):
    """A reference config file's text -> the device run of its (or the given) method."""
    cfg = parse_config(text)
    return run_method_on(cfg, build_setup(cfg), method or cfg.method, device)


# ----------------------------------------------------------------------------------- reports
@dataclass
class ReportRow:  # harness.hpp ReportRow
    label: str
    m: float
    amt: float
    speedup: float
    hit_rate: float
    tokens: int
    clock: float


def _row(label, res) -> ReportRow:  # row_from, harness.cpp:389-399
    mt = res.metrics
    return ReportRow(label, mt["m"], mt["amt"], mt["speedup"], mt["hit_rate"], int(mt["tokens"]), mt["clock"])


def run_pipelined(cfg: ExperimentConfig, setup: ExperimentSetup, draft_retrieval: bool, target_retrieval: bool,
                  rejected_cache: bool, device: int = 0):
    """run_pipelined (harness.cpp:371-387) on the device."""
    st = HierarchicalDatastore(cfg.ngram, cfg.depth, device)
    for i, seq in enumerate(setup.corpus[:cfg.prior_rounds]):
        st.prior.insert(seq, i)
    st.rejected_enabled = rejected_cache
    opts = PipelineOptions(gamma=cfg.effective_gamma(), depth=cfg.depth, draft_retrieval=draft_retrieval,
                           target_retrieval=target_retrieval, t_target=cfg.t_target, t_draft=cfg.t_draft,
                           t_lookup=cfg.t_lookup, t_sync=cfg.t_sync, temperature=cfg.temperature,
                           rng_seed=cfg.seed, engine=cfg.engine)
    return run(setup.draft.device(device), setup.target.device(device), st, setup.prompt, cfg.max_new_tokens, opts)
