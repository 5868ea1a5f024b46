"""Batched-serving throughput: run_vanilla_ar_batch for B sequences of the bench workload's shape."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2601_05524_b200 as dbl  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "qwen3-14b"
n_new = int(sys.argv[2]) if len(sys.argv) > 2 else 64
m = dbl.Transformer(dbl.transformer_config(name, seed=1, max_seq=4096))
for B in (1, 2, 4, 8, 16):
    prompts = [bench.workload(m.cfg.vocab, 160, 300 + b)[0] for b in range(B)]
    dbl.run_vanilla_ar_batch(m, prompts, 4)  # warm-up
    outs, met = dbl.run_vanilla_ar_batch(m, prompts, n_new)
    print(f"{name} B={B:2d} tokens={met['tokens']:5d} loop={met['device_ms']:.1f} ms "
          f"-> {met['tokens'] / met['device_ms'] * 1e3:.1f} tok/s ({met['device_ms'] / n_new:.3f} ms/step)")

# batched DOUBLE (draft + target, one datastore per sequence)
if len(sys.argv) > 3 and sys.argv[3] == "double":
    drf = dbl.Transformer(dbl.transformer_config("qwen3-0.6b", seed=2, max_seq=4096))
    for B in (1, 4, 8, 16):
        ps, pr = [], []
        for b in range(B):
            p, prior = bench.workload(m.cfg.vocab, 160, 300 + b)
            ps.append(p)
            pr.append(prior)

        def stores():
            out = []
            for b in range(B):
                st = dbl.HierarchicalDatastore(3, 10)
                dbl.build_prior(st, pr[b], 10)
                out.append(st)
            return out
        o = dbl.PipelineOptions(gamma=1, depth=10)
        dbl.run_batch(drf, m, stores(), ps, 8, o, want_jsonl=False)
        rs = dbl.run_batch(drf, m, stores(), ps, n_new, o, want_jsonl=False)
        toks = sum(len(r.output) for r in rs)
        ms = rs[0].metrics["device_ms"]
        print(f"double B={B:2d} tokens={toks:5d} loop={ms:.1f} ms -> {toks / ms * 1e3:.1f} tok/s")
