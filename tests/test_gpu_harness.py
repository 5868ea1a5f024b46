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


def test_acceptance_criteria_5_to_7_on_device(hz):
    """The reference's acceptance gate (acceptance.cpp:214-299) with every decode on the device:
    5 — Double breaks the PSD ceiling C on the shipped config; 6 — each component helps (ablation);
    7 — M is monotone in the retrieval depth and saturates from d=10 to d=20."""
    import dataclasses
    cfg = hz.parse_config(CFG1["config"])
    s = hz.build_setup(cfg)
    c = cfg.t_target / cfg.t_draft
    dbl_row = hz._row("double", hz.run_method_on(cfg, s, "double"))
    psd_row = hz._row("psd", hz.run_method_on(cfg, s, "psd"))
    assert dbl_row.speedup > c and psd_row.speedup <= c + 1e-9
    a = hz.ExperimentConfig(vocab=32, rho=0.8, corpus_len=4096, draft_order=1, target_order=2, t_target=1.0,
                            t_draft=0.625, gamma=2, depth=10, prior_rounds=0, max_new_tokens=512, seed=44)
    rows = hz.ablate(a)
    full, wo_draft, wo_target, wo_rejected = rows[:4]
    assert full.m > wo_target.m and full.speedup > wo_draft.speedup and full.hit_rate > wo_rejected.hit_rate
    assert "wo_prior" in hz.emit_report(rows) and hz.emit_report(rows, "csv").startswith("method,m,amt")
    sw = hz.ExperimentConfig(vocab=32, rho=0.95, corpus_len=4096, draft_order=1, target_order=2, t_target=1.0,
                             t_draft=0.625, gamma=0, max_new_tokens=256)
    for seed in (3, 7, 11, 17):
        ms = [r.m for r in hz.sweep_depth(dataclasses.replace(sw, seed=seed), [1, 2, 4, 10, 20])]
        assert all(ms[i] >= ms[i - 1] - 1e-9 for i in range(1, len(ms))), (seed, ms)
    sat = hz.sweep_depth(dataclasses.replace(sw, rho=0.7, t_draft=0.25, gamma=4, seed=11), [10, 20])
    assert (sat[1].m - sat[0].m) / sat[0].m < 0.05


def test_cli_run_writes_the_reference_trace(tmp_path):
    import subprocess
    import sys
    from conftest import ROOT
    cfg = tmp_path / "ceiling_break.cfg"
    cfg.write_text(CFG1["config"])
    tr = tmp_path / "trace.jsonl"
    r = subprocess.run([sys.executable, "-m", "paper_2601_05524_b200", "run", "--config", str(cfg), "--trace", str(tr)],
                       env=dict(os.environ, PYTHONPATH=ROOT), capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert hashlib.sha256(tr.read_text().encode()).hexdigest() == CFG1["methods"]["double"]["jsonl_sha256"]
    assert "double" in r.stdout and "speedup" in r.stdout
