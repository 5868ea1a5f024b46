"""Repeat the same DOUBLE decode (bench workload shapes, gamma 1 = the half-grid draft beside the verify,
and gamma 4 = full grid) and check every run's output and JSONL are identical, and equal target-only AR.
    python tools/decode_determinism.py [reps] [max_new]"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_05524_b200 as dbl  # noqa: E402
from bench import workload, DEPTH, NGRAM, PRIOR_K  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
max_new = int(sys.argv[2]) if len(sys.argv) > 2 else 128
tgt = dbl.Transformer(dbl.transformer_config("qwen3-14b", seed=1, max_seq=4096, n_layers=4))
drf = dbl.Transformer(dbl.transformer_config("qwen3-0.6b", seed=2, max_seq=4096))
prompt, prior = workload(tgt.cfg.vocab, 900, 101)
ar = dbl.run_vanilla_ar(tgt, prompt, max_new).output
for g in (1, 4):
    outs, js = set(), set()
    for _ in range(reps):
        st = dbl.HierarchicalDatastore(NGRAM, DEPTH)
        dbl.build_prior(st, prior, PRIOR_K)
        r = dbl.run(drf, tgt, st, prompt, max_new, dbl.PipelineOptions(gamma=g, depth=DEPTH))
        outs.add(tuple(r.output))
        js.add(hashlib.sha256(r.jsonl.encode()).hexdigest())
    print(f"gamma {g}: {reps} decodes, {len(outs)} distinct outputs, {len(js)} distinct JSONL, "
          f"== AR: {list(outs)[0] == tuple(ar) if len(outs) == 1 else False}", flush=True)
