"""Small device workload for compute-sanitizer (memcheck / racecheck / synccheck): the table-model
DOUBLE loop greedy and sampled, serial SD and AR sampled, retrieval kernels and the verifier API.
(The persistent transformer forward is excluded: its spin-waits + 4 s watchdog do not survive the
sanitizer's slowdown.)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2601_05524_b200 as dbl  # noqa: E402
from paper_2601_05524_b200.specpar import parse_dstore_v1  # noqa: E402

G = os.path.join(ROOT, "tests", "golden")
d = dbl.TableModel.from_model_v1(open(os.path.join(G, "config1_draft.model-v1")).read())
t = dbl.TableModel.from_model_v1(open(os.path.join(G, "config1_target.model-v1")).read())
_, seqs = parse_dstore_v1(open(os.path.join(G, "config1_prior.dstore-v1")).read())
prompt = json.load(open(os.path.join(G, "config1.json")))["prompt"]
for temp in (0.0, 1.0, 0.7):
    st = dbl.HierarchicalDatastore(3, 10)
    dbl.build_prior(st, seqs, len(seqs))
    o = dbl.PipelineOptions(gamma=2, depth=10, t_draft=0.625, temperature=temp, rng_seed=11)
    r = dbl.run(d, t, st, prompt, 48, o)
    st2 = dbl.HierarchicalDatastore(3, 10)
    dbl.build_prior(st2, seqs, len(seqs))
    s = dbl.run_serial_sd(d, t, st2, prompt, 32, o, use_retrieval=True)
    a = dbl.run_vanilla_ar(t, prompt, 32, temperature=temp, rng_seed=11)
    print(temp, len(r.output), len(s.output), len(a.output))
rng = dbl.Rng(5)
p = np.array([0.1, 0.2, 0.7]); q = np.array([0.3, 0.3, 0.4])
print(dbl.specpar.accept_prob(p, q, 2), dbl.specpar.residual_sample(p, q, rng))
print("ok")
