"""GPU: batched serving — several independent sequences share ONE verify forward
(fwd_kernel<kB>: per-row lane, position, page table and KV cache).  Every sequence's greedy stream
equals its own single-sequence run_vanilla_ar bitwise: a row's arithmetic never depends on the other
rows (the batch-invariance argument of the single-lane forward, extended across sequences)."""
import random

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dbl():
    import paper_2601_05524_b200 as dbl
    assert dbl._capi.lib().dbl_device_ok() == 1
    return dbl


@pytest.mark.parametrize("name,B,lens,n", [("tiny-qwen", 4, (5, 17, 64, 100), 48),
                                           ("tiny-llama", 16, None, 24)])
def test_batched_ar_equals_single_sequence_ar(dbl, name, B, lens, n):
    cfg = dbl.transformer_config(name, seed=7, max_seq=2048)
    m = dbl.Transformer(cfg)
    rng = random.Random(B)
    lens = lens or [rng.randint(1, 300) for _ in range(B)]
    prompts = [[rng.randrange(1, cfg.vocab - 1) for _ in range(L)] for L in lens]
    outs, met = dbl.run_vanilla_ar_batch(m, prompts, n)
    assert len(outs) == B
    for p, o in zip(prompts, outs):
        assert o == dbl.run_vanilla_ar(m, p, n).output
    assert met["tokens"] == sum(len(o) for o in outs)


def test_batched_ar_limits(dbl):
    m = dbl.Transformer(dbl.transformer_config("tiny-qwen", seed=1, max_seq=512))
    with pytest.raises(dbl.InvalidArgument):
        dbl.run_vanilla_ar_batch(m, [[1, 2]] * 17, 4)
    with pytest.raises(dbl.InvalidArgument):
        dbl.run_vanilla_ar_batch(m, [[1, 2], []], 4)


KEYS = ("tokens", "rounds", "clock", "m", "amt", "speedup", "hit_rate", "lookups")


def _prior(vocab, seed, n=6):
    rng = random.Random(seed)
    base = [rng.randrange(1, vocab - 1) for _ in range(40)]
    out = []
    for _ in range(n):
        s = []
        while len(s) < 48:
            s += base[rng.randrange(0, 30):][: rng.randrange(4, 12)] if rng.random() < 0.7 else \
                [rng.randrange(1, vocab - 1) for _ in range(3)]
        out.append(s[:48])
    return out


def _check_batch_equals_single(dbl, drf, tgt, prior, prompts, n, opts):
    def store():
        st = dbl.HierarchicalDatastore(3, opts.depth)
        dbl.build_prior(st, prior, len(prior))
        return st
    batch = dbl.run_batch(drf, tgt, [store() for _ in prompts], prompts, n, opts)
    for p, r in zip(prompts, batch):
        one = dbl.run(drf, tgt, store(), p, n, opts)
        assert r.output == one.output
        assert r.jsonl == one.jsonl
        assert [r.metrics[k] for k in KEYS] == [one.metrics[k] for k in KEYS]


def test_batched_double_equals_single_runs_tables(dbl):
    import json
    import os
    from conftest import GOLDEN
    from paper_2601_05524_b200.specpar import parse_dstore_v1
    d = dbl.TableModel.from_model_v1(open(os.path.join(GOLDEN, "config1_draft.model-v1")).read())
    t = dbl.TableModel.from_model_v1(open(os.path.join(GOLDEN, "config1_target.model-v1")).read())
    _, seqs = parse_dstore_v1(open(os.path.join(GOLDEN, "config1_prior.dstore-v1")).read())
    base = json.load(open(os.path.join(GOLDEN, "config1.json")))["prompt"]
    prompts = [base, base[:5], seqs[3][:12], seqs[7][:3]]
    _check_batch_equals_single(dbl, d, t, seqs, prompts, 96,
                               dbl.PipelineOptions(gamma=2, depth=10, t_draft=0.625))


@pytest.mark.parametrize("gamma", [1, 3])
def test_batched_double_equals_single_runs_transformers(dbl, gamma):
    tgt = dbl.Transformer(dbl.transformer_config("tiny-qwen", seed=11, max_seq=2048))
    drf = dbl.Transformer(dbl.transformer_config("tiny-qwen-draft", seed=12, max_seq=2048))
    prior = _prior(tgt.cfg.vocab, 4)
    prompts = [prior[0][:24], prior[1][:9], prior[2][:40], [5, 6, 7]]
    _check_batch_equals_single(dbl, drf, tgt, prior, prompts, 64, dbl.PipelineOptions(gamma=gamma, depth=10))


def test_batched_double_limits(dbl):
    tgt = dbl.Transformer(dbl.transformer_config("tiny-qwen", seed=1, max_seq=512))
    st = dbl.HierarchicalDatastore(3, 10)
    with pytest.raises(dbl.InvalidArgument):  # one datastore per sequence
        dbl.run_batch(tgt, tgt, [st, st], [[1, 2], [3, 4]], 4)


@pytest.mark.parametrize("temperature", [1.0, 0.8])
def test_batched_sampled_double_equals_single_runs(dbl, temperature):
    """T > 0: every sequence of the batch draws its own derive_rng streams, so each equals its own
    sampled run (distribution rows from one batched forward + per-lane softmax)."""
    tgt = dbl.Transformer(dbl.transformer_config("tiny-qwen", seed=21, max_seq=2048, init_std=0.08))
    drf = dbl.Transformer(dbl.transformer_config("tiny-qwen-draft", seed=22, max_seq=2048, init_std=0.08))
    prior = _prior(tgt.cfg.vocab, 6)
    prompts = [prior[0][:20], prior[3][:7], [9, 8, 7, 6]]
    _check_batch_equals_single(dbl, drf, tgt, prior, prompts, 48,
                               dbl.PipelineOptions(gamma=2, depth=8, temperature=temperature, rng_seed=77))
