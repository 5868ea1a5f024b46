"""Wall-clock breakdown of one public run() call at the bench workload (host overhead hunting)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2601_05524_b200 as dbl  # noqa: E402

name_t = sys.argv[1] if len(sys.argv) > 1 else "qwen3-14b"
name_d = sys.argv[2] if len(sys.argv) > 2 else "qwen3-0.6b"
tgt = dbl.Transformer(dbl.transformer_config(name_t, seed=1, max_seq=4096))
drf = dbl.Transformer(dbl.transformer_config(name_d, seed=2, max_seq=4096))
prompt, prior = bench.workload(tgt.cfg.vocab, 160, 101)
print("prior seqs", len(prior), "lens", [len(s) for s in prior][:12])
opts = dbl.PipelineOptions(gamma=1, depth=bench.DEPTH)
for it in range(3):
    t0 = time.perf_counter()
    st = dbl.HierarchicalDatastore(bench.NGRAM, bench.DEPTH)
    t1 = time.perf_counter()
    dbl.build_prior(st, prior, bench.PRIOR_K)
    t2 = time.perf_counter()
    r = dbl.run(drf, tgt, st, prompt, 256, opts, want_jsonl=False)
    t3 = time.perf_counter()
    m = r.metrics
    print(f"store {1e3*(t1-t0):.1f} ms prior {1e3*(t2-t1):.1f} ms run {1e3*(t3-t2):.1f} ms "
          f"(device {m['device_ms']:.1f} prefill {m['prefill_ms']:.1f}) tokens {len(r.output)}")
