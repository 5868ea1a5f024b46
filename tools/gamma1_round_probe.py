"""gamma = 1 DOUBLE decodes of the bench workload: device ms per round vs the verify forward (cooperative
vs plain launches with DBL_FWD_COOP=0)."""
import os, sys, json
sys.path.insert(0, os.getcwd())
import paper_2601_05524_b200 as dbl
from bench import WORKLOADS, workload, DEPTH, NGRAM, PRIOR_K
tgt = dbl.Transformer(dbl.transformer_config("qwen3-14b", seed=1, max_seq=4096))
drf = dbl.Transformer(dbl.transformer_config("qwen3-0.6b", seed=2, max_seq=4096))
prompt, prior = workload(tgt.cfg.vocab, 160, 101)
for n in (128, 256, 256, 256):
    st = dbl.HierarchicalDatastore(NGRAM, DEPTH); dbl.build_prior(st, prior, PRIOR_K)
    r = dbl.run(drf, tgt, st, prompt, n, dbl.PipelineOptions(gamma=1, depth=DEPTH), want_jsonl=False)
    m = r.metrics
    print(n, m["rounds"], round(m["device_ms"], 1), round(m["device_ms"] / m["rounds"], 3), "tok/s", round(len(r.output) / m["device_ms"] * 1e3, 1), "verify", round(m["target_fwd_ms"] / m["target_fwd_count"], 3))
