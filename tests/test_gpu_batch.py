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
