"""Cost of the sampled (T > 0) loop vs greedy on the bench workload shapes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2601_05524_b200 as dbl  # noqa: E402

tgt = dbl.Transformer(dbl.transformer_config("qwen3-14b", seed=1, max_seq=4096))
drf = dbl.Transformer(dbl.transformer_config("qwen3-0.6b", seed=2, max_seq=4096))
prompt, prior = bench.workload(tgt.cfg.vocab, 160, 101)
for T in (0.0, 1.0, 0.7):
    for it in range(2):
        st = dbl.HierarchicalDatastore(3, 10)
        dbl.build_prior(st, prior, 10)
        r = dbl.run(drf, tgt, st, prompt, 64, dbl.PipelineOptions(gamma=1, depth=10, temperature=T, rng_seed=3),
                    want_jsonl=False)
        a = dbl.run_vanilla_ar(tgt, prompt, 64, temperature=T, rng_seed=3, want_jsonl=False)
    m = r.metrics
    print(f"T={T}: DOUBLE {len(r.output) / m['device_ms'] * 1e3:.1f} tok/s ({m['device_ms'] / m['rounds']:.2f} ms/round, "
          f"target fwd {m['target_fwd_ms'] / m['target_fwd_count']:.2f} ms)  AR {len(a.output) / a.metrics['device_ms'] * 1e3:.1f} tok/s")
