import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2601_05524_b200 as dbl  # noqa: E402
tgt = dbl.Transformer(dbl.transformer_config("qwen3-14b", seed=1, max_seq=4096))
drf = dbl.Transformer(dbl.transformer_config("qwen3-0.6b", seed=2, max_seq=4096))
prompt, prior = bench.workload(tgt.cfg.vocab, 160, 101)
st = dbl.HierarchicalDatastore(3, 10)
dbl.build_prior(st, prior, 10)
r = dbl.run(drf, tgt, st, prompt, 8, dbl.PipelineOptions(gamma=1, depth=10, temperature=float(sys.argv[1]), rng_seed=3), want_jsonl=False)
print(len(r.output))
