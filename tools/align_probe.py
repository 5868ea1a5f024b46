"""How often does a draft agree with the random-init target (teacher-forced, greedy)?  Candidate
aligned drafts for a labelled alpha > 0 workload (SURVEY §7 hard part 6): early-exit drafts (the
target's own first k layers + its embedding / LM head, same seed).
    python tools/align_probe.py [target] [n_tokens]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_05524_b200 as dbl  # noqa: E402
from bench import workload  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "qwen3-14b"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
for spec in (sys.argv[3] if len(sys.argv) > 3 else "0:1,1:0.1").split(","):
    k0, scale = int(spec.split(":")[0]), float(spec.split(":")[1])
    kw = dict(layer_std_scale=scale, scale_from_layer=k0)
    tgt = dbl.Transformer(dbl.transformer_config(name, seed=1, max_seq=2048, **kw))
    prompt, _ = workload(tgt.cfg.vocab, 160, 101)
    ar = dbl.run_vanilla_ar(tgt, prompt, n, want_jsonl=False).output
    print(f"{name} layers >= {k0} x{scale}: {len(ar)} AR tokens, {len(set(ar))} distinct; head {ar[:12]}")
    del tgt
    for k in sorted({max(1, k0), k0 + 1, 4}):
        d = dbl.Transformer(dbl.transformer_config(name, seed=1, max_seq=2048, n_layers=k, **kw))
        rows = dbl.forward_batch(d, prompt, ar[:n - 1])
        agree = sum(int(a == b) for a, b in zip(rows, ar)) / len(ar)
        st = dbl.HierarchicalDatastore(3, 10)
        print(f"  early-exit {k} layers: alpha={agree:.3f}  weight GB={d.weight_bytes / 1e9:.2f}")
        del d
