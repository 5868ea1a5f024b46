"""Is the draft's forward concurrent with the verify forward?  gamma = 1 decodes of the bench workload
with and without the round timeline's CUDA events, and with the draft's stream work held back until the
target's forward has been launched (DBL_TARGET_FIRST=1)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import os, sys
sys.path.insert(0, %r)
import paper_2601_05524_b200 as dbl
from bench import WORKLOADS, workload, DEPTH, NGRAM, PRIOR_K
tgt = dbl.Transformer(dbl.transformer_config("qwen3-14b", seed=1, max_seq=4096))
drf = dbl.Transformer(dbl.transformer_config("qwen3-0.6b", seed=2, max_seq=4096))
prompt, prior = workload(tgt.cfg.vocab, 160, 101)
res = []
for g in (1, 1, 2):
    st = dbl.HierarchicalDatastore(NGRAM, DEPTH); dbl.build_prior(st, prior, PRIOR_K)
    r = dbl.run(drf, tgt, st, prompt, 128, dbl.PipelineOptions(gamma=g, depth=DEPTH), want_jsonl=False)
    res.append((g, r.metrics["device_ms"] / r.metrics["rounds"], r.metrics["target_fwd_ms"] / max(1, r.metrics["target_fwd_count"])))
ar = dbl.run_vanilla_ar(tgt, prompt, 64, want_jsonl=False)
print(os.environ.get("TAG"), " ".join(f"g{g}: {a:.3f} ms/round (verify {b:.3f})" for g, a, b in res), f"AR {ar.metrics['device_ms']/64:.3f} ms/token")
''' % ROOT
for tag, env in (("plain", {}), ("timeline", {"DBL_ROUND_TIMELINE_FILE": "/tmp/tl.jsonl", "DBL_ROUND_TIMELINE_N": "1000"}),
                 ("target_first", {"DBL_TARGET_FIRST": "1"})):
    e = dict(os.environ, TAG=tag, **env)
    r = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True)
    print(r.stdout.strip() or r.stderr[-500:], flush=True)
