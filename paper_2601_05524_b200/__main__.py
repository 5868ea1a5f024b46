"""Command line mirroring the reference's `specpar` tool (tools/specpar_main.cpp) for the decode-path
subcommands, every decode on the device:

    python -m paper_2601_05524_b200 run --config proj/configs/ceiling_break.cfg [--trace t.jsonl]
                                        [--report r.txt --format text|csv]
    python -m paper_2601_05524_b200 ablate --config C [--out F --format text|csv]
    python -m paper_2601_05524_b200 sweep-depth --config C --depths 1,2,4,10,20 [--out F --format ...]
    python -m paper_2601_05524_b200 gen-corpus --vocab 32 --rho 0.5 --length 4096 --seed 1 --out corpus.txt
    python -m paper_2601_05524_b200 build-prior --corpus corpus.txt --ngram 3 --rounds 10 --out prior.dstore

SPECPAR_SEED overrides the config's seed (specpar_main.cpp:40-44).  The closed-form `sweep` / `analyze`
subcommands (analytics.cpp) are outside the decode path and not mirrored."""
from __future__ import annotations

import argparse
import os
import sys

from . import harness
from .specpar import serialize_index


def _cfg(path):
    cfg = harness.load_config(path)
    if os.environ.get("SPECPAR_SEED"):  # apply_seed_override
        cfg.seed = int(os.environ["SPECPAR_SEED"])
    return cfg


def _write_report(rows, cfg, path, fmt):  # write_report, harness.cpp:502-515
    with open(path, "w") as f:
        if fmt == "text":
            f.write("".join("# " + ln + "\n" for ln in harness.serialize_config(cfg).splitlines()))
        f.write(harness.emit_report(rows, fmt))


def main(argv=None) -> int:
    p = argparse.ArgumentParser(prog="paper_2601_05524_b200")
    sub = p.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("gen-corpus")
    g.add_argument("--vocab", type=int, default=32)
    g.add_argument("--rho", type=float, default=0.5)
    g.add_argument("--length", type=int, default=4096)
    g.add_argument("--seed", type=int, default=1)
    g.add_argument("--out", default="corpus.txt")
    b = sub.add_parser("build-prior")
    b.add_argument("--corpus", required=True)
    b.add_argument("--ngram", type=int, default=3)
    b.add_argument("--rounds", type=int, default=10)
    b.add_argument("--out", default="prior.dstore")
    r = sub.add_parser("run")
    r.add_argument("--config", required=True)
    r.add_argument("--trace", default="")
    r.add_argument("--report", default="")
    r.add_argument("--format", default="text")
    a = sub.add_parser("ablate")
    a.add_argument("--config", required=True)
    a.add_argument("--out", default="")
    a.add_argument("--format", default="text")
    d = sub.add_parser("sweep-depth")
    d.add_argument("--config", required=True)
    d.add_argument("--depths", default="1,2,4,10,20")
    d.add_argument("--out", default="")
    d.add_argument("--format", default="text")
    args = p.parse_args(argv)
    try:
        if args.cmd == "gen-corpus":
            corpus = harness.gen_corpus(args.vocab, args.rho, args.length, args.seed)
            with open(args.out, "w") as f:  # save_corpus_lines
                f.write("".join(" ".join(map(str, s)) + "\n" for s in corpus))
            print(f"wrote {args.out}")
        elif args.cmd == "build-prior":
            with open(args.corpus) as f:  # load_corpus_lines
                corpus = [[int(t) for t in ln.split()] for ln in f if ln.split()]
            with open(args.out, "w") as f:  # build_prior + save_index
                f.write(serialize_index(args.ngram, corpus[:max(0, args.rounds)]))
            print(f"wrote {args.out}")
        elif args.cmd == "run":
            cfg = _cfg(args.config)
            res = harness.run_method_on(cfg, harness.build_setup(cfg), cfg.method)
            row = harness._row(cfg.method, res)
            if args.trace:
                with open(args.trace, "w") as f:  # write_traces
                    f.write(res.jsonl)
            sys.stdout.write(harness.emit_report([row], "text"))
            if args.report:
                _write_report([row], cfg, args.report, args.format)
        elif args.cmd == "ablate":
            cfg = _cfg(args.config)
            rows = harness.ablate(cfg)
            sys.stdout.write(harness.emit_report(rows, "text"))
            if args.out:
                _write_report(rows, cfg, args.out, args.format)
        elif args.cmd == "sweep-depth":
            cfg = _cfg(args.config)
            rows = harness.sweep_depth(cfg, [int(x) for x in args.depths.split(",") if x])
            sys.stdout.write(harness.emit_report(rows, "text"))
            if args.out:
                _write_report(rows, cfg, args.out, args.format)
    except Exception as e:  # noqa: BLE001 — the reference prints "error: ..." and exits 1
        print(f"error: {e}", file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
