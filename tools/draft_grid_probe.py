"""DOUBLE decode rate on one GPU vs the draft's grid (DBL_DRAFT_GRID_DIV: the draft's forward on 1/k of
the SMs, launched plainly beside the verify's cooperative grid): both bench workloads, gamma 1 / 4 / 8."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_05524_b200 as dbl  # noqa: E402
from bench import WORKLOADS, workload, DEPTH, NGRAM, PRIOR_K  # noqa: E402

for name in ("qwen3-0.6b/qwen3-14b", "aligned-qwen3-14b"):
    wl = WORKLOADS[name]
    (tn, tkw), (dn, dkw) = wl["target"], wl["draft"]
    tgt = dbl.Transformer(dbl.transformer_config(tn, seed=1, max_seq=4096, **tkw))
    drf = dbl.Transformer(dbl.transformer_config(dn, seed=1 if wl.get("same_seed") else 2, max_seq=4096, **dkw))
    prompt, prior = workload(tgt.cfg.vocab, wl["prompt_len"], 101)
    res = []
    for g in (1, 4, 8):
        best = 0.0
        for _ in range(2):
            st = dbl.HierarchicalDatastore(NGRAM, DEPTH)
            dbl.build_prior(st, prior, PRIOR_K)
            r = dbl.run(drf, tgt, st, prompt, 256, dbl.PipelineOptions(gamma=g, depth=DEPTH), want_jsonl=False)
            best = max(best, len(r.output) / r.metrics["device_ms"] * 1e3)
        res.append(f"g{g} {best:.1f}")
    print(f"div={os.environ.get('DBL_DRAFT_GRID_DIV', '1')} {name}: " + "  ".join(res), flush=True)
    del tgt, drf
