"""compute-sanitizer workload for the persistent transformer forward (fwd_kernel): tiny-qwen (2 layers,
h=256, V=1024) forward_batch at 1 / 5 / 20 rows and one short DOUBLE decode.  The watchdog is lengthened
(DBL_FWD_WATCHDOG_MS) so the sanitizer's slowdown is not mistaken for a stalled dependency."""
import os
import sys

os.environ.setdefault("DBL_FWD_WATCHDOG_MS", "600000")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_05524_b200 as dbl  # noqa: E402

m = dbl.Transformer(dbl.transformer_config("tiny-qwen", seed=3, max_seq=512))
d = dbl.Transformer(dbl.transformer_config("tiny-qwen-draft", seed=4, max_seq=512))
ctx = [(7 * i + 3) % 1000 + 1 for i in range(70)]
for c in (0, 4, 19):
    print("rows", c + 1, dbl.forward_batch(m, ctx, ctx[5:5 + c])[:4])
r = dbl.run(d, m, dbl.HierarchicalDatastore(3, 10), ctx[:30], 12, dbl.PipelineOptions(gamma=2))
print("double", r.output)
print("ok")
