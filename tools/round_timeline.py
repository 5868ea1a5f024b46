"""PSD draft-while-verify on one GPU, as a device timeline: runs the bench workloads with
DBL_ROUND_TIMELINE_FILE set (decoder.cu DoubleEngine::Timeline) and summarises, per gamma, how much of
the draft chain overlaps the verify forward.

    python tools/round_timeline.py [out.jsonl]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
path = sys.argv[1] if len(sys.argv) > 1 else "/tmp/round_timeline.jsonl"
if os.path.exists(path):
    os.remove(path)
os.environ["DBL_ROUND_TIMELINE_FILE"] = path
os.environ["DBL_ROUND_TIMELINE_N"] = "40"
import paper_2601_05524_b200 as dbl  # noqa: E402
from bench import WORKLOADS, workload, DEPTH, NGRAM, PRIOR_K  # noqa: E402


def decode(wl_name, gammas):
    wl = WORKLOADS[wl_name]
    (tn, tkw), (dn, dkw) = wl["target"], wl["draft"]
    tgt = dbl.Transformer(dbl.transformer_config(tn, seed=1, max_seq=4096, **tkw))
    drf = dbl.Transformer(dbl.transformer_config(dn, seed=1 if wl.get("same_seed") else 2, max_seq=4096, **dkw))
    prompt, prior = workload(tgt.cfg.vocab, wl["prompt_len"], 101)
    out = {}
    for g in gammas:
        st = dbl.HierarchicalDatastore(NGRAM, DEPTH)
        dbl.build_prior(st, prior, PRIOR_K)
        n0 = sum(1 for _ in open(path)) if os.path.exists(path) else 0
        r = dbl.run(drf, tgt, st, prompt, 96, dbl.PipelineOptions(gamma=g, depth=DEPTH), want_jsonl=False)
        rows = [json.loads(x) for x in open(path)][n0:]
        out[g] = (rows, r.metrics)
    del tgt, drf
    return out


def summarise(name, res):
    print(f"== {name}")
    for g, (rows, m) in res.items():
        rows = rows[2:]  # skip the first rounds (lane caches, L2 warm-up)
        tf = [r["target_fwd"][1] - r["target_fwd"][0] for r in rows]
        dr = [sum(e - s for s, e in r["draft"]) for r in rows]
        ov = []
        for r in rows:
            a, b = r["target_fwd"]
            ov.append(sum(max(0.0, min(e, b) - max(s, a)) for s, e in r["draft"]))
        span = [max(r["target_end"], max(e for _, e in r["draft"])) for r in rows]
        hw = [r["host_wait_us"] for r in rows]
        hf = [r["host_finish_us"] for r in rows]
        avg = lambda v: sum(v) / max(1, len(v))  # noqa: E731
        print(f"  gamma {g}: {len(rows)} rounds; verify fwd {avg(tf):.0f} us ({avg([r['target_rows'] for r in rows]):.1f} rows), "
              f"draft chain {avg(dr):.0f} us of which {avg(ov):.0f} us under the verify forward "
              f"({100 * avg(ov) / max(1e-9, avg(dr)):.0f} %); device span {avg(span):.0f} us; host wait {avg(hw):.0f} us, "
              f"host finish_round {avg(hf):.0f} us; decode {m['tokens'] / (m['device_ms'] / 1e3):.1f} tok/s, M {m['m']:.2f}")
        r = rows[len(rows) // 2]
        print(f"    e.g. round {r['round']}: verify [{r['target_fwd'][0]:.0f}, {r['target_fwd'][1]:.0f}] us, draft segments "
              + ", ".join(f"[{s:.0f}, {e:.0f}]" for s, e in r["draft"]))


summarise("qwen3-0.6b/qwen3-14b (configs[1], independent draft)", decode("qwen3-0.6b/qwen3-14b", [1, 4]))
summarise("aligned-qwen3-14b (labelled aligned workload)", decode("aligned-qwen3-14b", [4, 8, 16]))
