"""`cltk price` on the GPU.

    python -m paper_2108_03076_b200 price KERNEL --model MODEL.json [--paths N]
        [--seed S] [--at D ...] [--threads T] [--tenv TENV.json] [--rng philox|sobol]
        [--jit 0|1|auto] [--device D] [--devices D0,D1,...]

Mirrors the reference CLI's `price` subcommand (proj/tools/cli.cpp:155-162,
246-259): same options and defaults (paths 100000, seed 1, valuation day 0),
the same JSON result array on stdout (priceResultToJson, proj/src/pricing.cpp:
161-167) and the same error convention ("error: <message>" on stderr, exit
code = ErrorCode).  KERNEL is the compiled kernel the reference emits
(`cltk emit --format kernel`, or the kernel JSON), since contract parsing and
compilation stay the reference's.
"""
from __future__ import annotations

import argparse
import json
import sys


def _price(args) -> int:
    import paper_2108_03076_b200 as E
    sys.setrecursionlimit(max(sys.getrecursionlimit(), 200000))
    kernel = E.load_kernel(args.kernel)
    with open(args.model) as f:
        model = f.read()
    tenv = None
    if args.tenv:
        with open(args.tenv) as f:
            tenv = json.load(f)
    days = args.at or [0]
    jit = {"0": False, "1": True, "auto": "auto"}[args.jit]
    devices = [int(d) for d in args.devices.split(",") if d.strip()] if args.devices else None
    res = E.price(kernel, model, args.paths, args.seed, days, tenv, threads=args.threads,
                  device=args.device, rng=args.rng, jit=jit, devices=devices)
    out = [{"price": r["price"], "stdError": r["std_error"], "paths": r["paths"],
            "seed": r["seed"], "valuationDay": r["valuation_day"]} for r in res]
    print(json.dumps(out, separators=(",", ":")))
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2108_03076_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("price", help="Monte Carlo price on the GPU")
    p.add_argument("kernel", help="compiled kernel (.kernel text or kernel JSON)")
    p.add_argument("--model", required=True)
    p.add_argument("--paths", type=int, default=100000)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--at", type=int, nargs="*", default=None, help="valuation days (default 0)")
    p.add_argument("--threads", type=int, default=0, help="accepted; results never depend on it")
    p.add_argument("--tenv")
    p.add_argument("--rng", default="philox", choices=["philox", "sobol"])
    p.add_argument("--jit", default="auto", choices=["0", "1", "auto"])
    p.add_argument("--device", type=int, default=-1)
    p.add_argument("--devices", default=None,
                   help="shard over these GPUs of this process (comma-separated; one NCCL "
                        "all-gather; the same bits as one GPU)")
    args = ap.parse_args(argv)
    try:
        return _price(args)
    except Exception as e:  # noqa: BLE001 -- the CLI's error convention
        code = getattr(e, "code", 5)
        print(f"error: {e}", file=sys.stderr)
        return int(code) if isinstance(code, int) else 5


if __name__ == "__main__":
    sys.exit(main())
