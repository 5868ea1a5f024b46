"""The draft on its own GPU (PSD draft-while-verify across devices, BASELINE configs 3-4; SURVEY
§8(e) "Draft placement"): the draft side then reads a replica of the datastore on its device that
receives finish_round's appends in the same order (SURVEY §8(b) threading).  DBL_STORE_MIRROR=1
forces that replica on one GPU, so the replication path is checked here against the same golden
vectors as the single-store loop; with >= 2 GPUs the draft also runs on device 1."""
import hashlib
import json
import os

import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu
CFG1 = json.load(open(os.path.join(GOLDEN, "config1.json")))


@pytest.fixture(scope="module")
def dbl():
    import paper_2601_05524_b200 as dbl
    assert dbl._capi.lib().dbl_device_ok() == 1, "no sm_100 device / library failed to load"
    return dbl


@pytest.fixture
def mirror():
    os.environ["DBL_STORE_MIRROR"] = "1"
    yield
    os.environ.pop("DBL_STORE_MIRROR", None)


def _cfg1(dbl, device=0):
    from paper_2601_05524_b200.specpar import parse_dstore_v1
    g = GOLDEN
    d = dbl.TableModel.from_model_v1(open(os.path.join(g, "config1_draft.model-v1")).read(), device=device)
    t = dbl.TableModel.from_model_v1(open(os.path.join(g, "config1_target.model-v1")).read())
    st = dbl.HierarchicalDatastore(3, 10)
    dbl.build_prior(st, parse_dstore_v1(open(os.path.join(g, "config1_prior.dstore-v1")).read())[1], 10)
    return d, t, st


@pytest.mark.parametrize("method", ["double", "psd", "target_retrieval"])
def test_config1_with_datastore_replica(dbl, mirror, method):
    d, t, st = _cfg1(dbl)
    want = CFG1["methods"][method]
    opts = dbl.PipelineOptions(gamma=2, depth=10, t_target=1.0, t_draft=0.625)
    opts.draft_retrieval = method == "double"
    opts.target_retrieval = method in ("double", "target_retrieval")
    r = dbl.run(d, t, st, CFG1["prompt"], 256, opts)
    assert r.output == want["output"]
    assert hashlib.sha256(r.jsonl.encode()).hexdigest() == want["jsonl_sha256"]
    m = want["metrics"]
    assert [r.metrics[k] for k in ("m", "amt", "hit_rate", "lookups")] == [m[k] for k in ("m", "amt", "hit_rate", "lookups")]
    # the replica's lookups were folded into the datastore's own stats; the session layers flushed
    s = st.stats
    assert s.lookups == m["lookups"]
    assert st.dynamic.occurrence_count() == 0 and st.rejected.occurrence_count() == 0


def test_transformer_with_datastore_replica(dbl, mirror):
    tgt = dbl.Transformer(dbl.transformer_config("tiny-qwen", seed=11, max_seq=1024))
    drf = dbl.Transformer(dbl.transformer_config("tiny-qwen-draft", seed=12, max_seq=1024))
    prompt = [(5 * i + 7) % 900 + 1 for i in range(40)]
    st = dbl.HierarchicalDatastore(3, 10)
    r = dbl.run(drf, tgt, st, prompt, 96, dbl.PipelineOptions(gamma=3, depth=10))
    os.environ.pop("DBL_STORE_MIRROR", None)
    st2 = dbl.HierarchicalDatastore(3, 10)
    r2 = dbl.run(drf, tgt, st2, prompt, 96, dbl.PipelineOptions(gamma=3, depth=10))
    assert r.output == r2.output == dbl.run_vanilla_ar(tgt, prompt, 96).output
    assert r.jsonl == r2.jsonl
    assert r.metrics["lookups"] == r2.metrics["lookups"] and r.metrics["hit_rate"] == r2.metrics["hit_rate"]


def _gpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.skipif("_gpus() < 2", reason="needs 2 GPUs (the draft on device 1)")
def test_draft_on_its_own_gpu(dbl):
    d, t, st = _cfg1(dbl, device=1)
    want = CFG1["methods"]["double"]
    r = dbl.run(d, t, st, CFG1["prompt"], 256, dbl.PipelineOptions(gamma=2, depth=10, t_target=1.0, t_draft=0.625))
    assert r.output == want["output"]
    assert hashlib.sha256(r.jsonl.encode()).hexdigest() == want["jsonl_sha256"]
    tgt = dbl.Transformer(dbl.transformer_config("tiny-qwen", seed=11, max_seq=1024), device=0)
    drf = dbl.Transformer(dbl.transformer_config("tiny-qwen-draft", seed=12, max_seq=1024), device=1)
    prompt = [(5 * i + 7) % 900 + 1 for i in range(40)]
    r = dbl.run(drf, tgt, dbl.HierarchicalDatastore(3, 10), prompt, 96, dbl.PipelineOptions(gamma=3, depth=10))
    assert r.output == dbl.run_vanilla_ar(tgt, prompt, 96).output
