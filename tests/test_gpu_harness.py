"""GPU: a reference config file run through the harness (harness.py) on the device reproduces the
unmodified reference's results for every method — greedy (config1.json) and sampled (sampled.json)."""
import hashlib
import json
import os

import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu
CFG1 = json.load(open(os.path.join(GOLDEN, "config1.json")))
SAMP = json.load(open(os.path.join(GOLDEN, "sampled.json")))
KEYS = ("tokens", "rounds", "clock", "m", "amt", "speedup", "hit_rate", "lookups")


@pytest.fixture(scope="module")
def hz():
    import paper_2601_05524_b200 as dbl
    assert dbl._capi.lib().dbl_device_ok() == 1
    from paper_2601_05524_b200 import harness
    return harness


@pytest.mark.parametrize("method", ["vanilla_ar", "sd", "psd", "target_retrieval", "draft_retrieval", "double"])
def test_reference_config_file_on_device(hz, method):
    want = CFG1["methods"][method]
    r = hz.run_config(CFG1["config"], method)
    assert r.output == want["output"]
    assert hashlib.sha256(r.jsonl.encode()).hexdigest() == want["jsonl_sha256"]
    assert [r.metrics[k] for k in KEYS] == [want["metrics"][k] for k in KEYS]
    case = SAMP["config1"][1]  # temperature 0.7
    text = CFG1["config"].replace("temperature=0", f"temperature={case['temperature']}")
    rs = hz.run_config(text, method)
    assert rs.output == case["methods"][method]["output"]
    assert hashlib.sha256(rs.jsonl.encode()).hexdigest() == case["methods"][method]["jsonl_sha256"]
