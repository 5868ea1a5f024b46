"""GPU: the tensor-parallel target — TP shards exchanging O/down partial tiles and the
vocab-parallel argmax inside fwd_kernel over peer memory.  On one B200 the shards co-reside (each
fwd_kernel takes at most half an SM), which exercises the same exchange protocol as NVLink peers.

* logits of the TP model == the unsharded model within the bf16/fp32 tolerance (the row-parallel
  partial sums change the fp32 summation order, so not bitwise);
* batch invariance inside TP (bitwise) — the lossless identity needs nothing more;
* DOUBLE with a TP target == target-only AR with the same TP target (bitwise greedy streams)."""
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ATOL_REL = 2e-2


@pytest.fixture(scope="module")
def dbl():
    import paper_2601_05524_b200 as dbl
    assert dbl._capi.lib().dbl_device_ok() == 1
    return dbl


@pytest.mark.parametrize("name,world", [("tiny-qwen", 2), ("tiny-llama", 2)])
def test_tp_logits_match_unsharded(dbl, name, world):
    cfg = dbl.transformer_config(name, seed=3, max_seq=2048)
    full = dbl.Transformer(cfg)
    tp = dbl.TpTransformer(dbl.transformer_config(name, seed=3, max_seq=2048), devices=[0] * world)
    rng = random.Random(5)
    agree = total = 0
    for L, c in ((1, 0), (9, 4), (70, 10), (300, 15)):
        ctx = [rng.randrange(cfg.vocab) for _ in range(L)]
        cands = [rng.randrange(cfg.vocab) for _ in range(c)]
        a = dbl.forward_logits(full, ctx, cands)
        b = dbl.forward_logits(tp, ctx, cands)
        assert np.abs(a - b).max() <= ATOL_REL * np.abs(a).max(), (L, c)
        am = dbl.forward_batch(tp, ctx, cands)
        assert am == b.argmax(axis=1).tolist()  # the in-kernel (max, lowest global id) combine
        agree += int(np.sum(a.argmax(axis=1) == b.argmax(axis=1)))
        total += c + 1
    assert agree >= 0.9 * total


def test_tp_batch_invariance(dbl):
    tp = dbl.TpTransformer(dbl.transformer_config("tiny-qwen", seed=5, max_seq=2048), devices=[0, 0])
    rng = random.Random(2)
    ctx = [rng.randrange(tp.cfg.vocab) for _ in range(70)]
    cands = [rng.randrange(tp.cfg.vocab) for _ in range(40)]
    batched = dbl.forward_logits(tp, ctx, cands)
    for k in (0, 1, 7, 16, 17, 33, 40):
        single = dbl.forward_logits(tp, ctx + cands[:k], [])
        assert np.array_equal(single[0], batched[k]), k


def _table_draft(dbl, vocab, seed):
    """an order-1 table draft over the target's vocabulary (short, non-persistent device kernels)"""
    rng = np.random.default_rng(seed)
    probs = rng.random((vocab, vocab)) ** 8  # peaked rows
    probs /= probs.sum(axis=1, keepdims=True)
    return dbl.TableModel(1, vocab, np.arange(vocab, dtype=np.int32), probs, np.full(vocab, 1.0 / vocab))


def test_double_with_tp_target_equals_tp_ar(dbl):
    """Lossless identity with a tensor-parallel target.  Both shards share this GPU, so the draft is a
    table model: at most two persistent forwards may co-run on one GPU (a target shard's and a
    transformer draft's) — the deployment layout (one target shard per GPU, draft beside one)."""
    tcfg = dbl.transformer_config("tiny-qwen", seed=11, max_seq=2048)
    tgt = dbl.TpTransformer(tcfg, devices=[0, 0])
    drf = _table_draft(dbl, tcfg.vocab, 12)
    rng = random.Random(4)
    base = [rng.randrange(1, tcfg.vocab - 1) for _ in range(40)]
    prior = [(base * 3)[i:i + 64] for i in range(0, 30, 3)]
    prompt = prior[0][:24]
    for gamma in (1, 4):
        st = dbl.HierarchicalDatastore(3, 10)
        dbl.build_prior(st, prior, 10)
        r = dbl.run(drf, tgt, st, prompt, 96, dbl.PipelineOptions(gamma=gamma, depth=10))
        ar = dbl.run_vanilla_ar(tgt, prompt, 96)
        assert r.output == ar.output


@pytest.mark.parametrize("world", [2, 4, 8])
def test_double_transformer_draft_with_tp_target(dbl, world):
    """A transformer draft beside a TP=2/4/8 target whose shards share this GPU: more than two
    persistent forwards cannot co-run, so the decoder runs both workers on one stream (same round
    results by construction, pipeline.cpp:239-261) — DOUBLE == target-only AR with the TP target."""
    tcfg = dbl.transformer_config("tiny-qwen", seed=13, max_seq=2048, n_kv_heads=8, n_heads=8)
    tgt = dbl.TpTransformer(tcfg, devices=[0] * world)
    drf = dbl.Transformer(dbl.transformer_config("tiny-qwen-draft", seed=14, max_seq=2048))
    rng = random.Random(world)
    base = [rng.randrange(1, tcfg.vocab - 1) for _ in range(40)]
    prior = [(base * 3)[i:i + 64] for i in range(0, 30, 3)]
    prompt = prior[0][:24]
    ar = dbl.run_vanilla_ar(tgt, prompt, 64)
    for gamma in (1, 3):
        st = dbl.HierarchicalDatastore(3, 10)
        dbl.build_prior(st, prior, 10)
        r = dbl.run(drf, tgt, st, prompt, 64, dbl.PipelineOptions(gamma=gamma, depth=10))
        assert r.output == ar.output, (world, gamma)
