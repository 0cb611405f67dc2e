"""A/B measurement of K2 build variants (development helper, not shipped).

Build here (cross-compile):   python tools/ab_variants.py build  NAME="-DFLAG=1 ..." ...
Run on the GPU box:           python tools/ab_variants.py run    NAME ... [-- bench args]

Each variant is the whole library built with extra nvcc flags into tools/_ab/<NAME>.so
(git-ignored; it travels to the box with the snapshot).  `run` times every variant with
the same short bench command, interleaved over several rounds, and prints K2's fraction of
the measured HBM peak per variant (median over rounds).
"""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
AB = os.path.join(ROOT, "tools", "_ab")
sys.path.insert(0, ROOT)


def build(specs):
    import __graft_entry__ as g

    os.makedirs(AB, exist_ok=True)
    for spec in specs:
        name, _, flags = spec.partition("=")
        g.build(extra=flags.split(), out=os.path.join(AB, f"{name}.so"))
        print("built", name, flags, flush=True)


def run(names, bench_args, rounds=3):
    res = {n: [] for n in names}
    for r in range(rounds):
        for n in names:
            env = dict(os.environ)
            if n != "base":
                env["KVMIX_LIB"] = os.path.join(AB, f"{n}.so")
            cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "10", "--warmup", "3", "--no-cpu-baseline",
                   "--no-e2e", "--no-k1", "--no-churn", *bench_args]
            p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=300)
            try:
                d = json.loads(p.stdout.strip().splitlines()[-1])
                res[n].append((d["roofline"]["frac"], d["value"], d.get("parity", {}).get("pass")))
                print(f"round {r} {n:16s} frac {d['roofline']['frac']:.4f} tok/s {d['value']:.1f} "
                      f"parity {d.get('parity', {}).get('pass')} err {d.get('parity', {}).get('max_abs_err')}", flush=True)
            except Exception:  # noqa: BLE001
                print(f"round {r} {n}: FAILED\n{p.stdout[-2000:]}\n{p.stderr[-3000:]}", flush=True)
    for n in names:
        if res[n]:
            print(f"{n:16s} median frac {statistics.median(x[0] for x in res[n]):.4f}  "
                  f"median tok/s {statistics.median(x[1] for x in res[n]):.1f}")


if __name__ == "__main__":
    mode, rest = sys.argv[1], sys.argv[2:]
    if mode == "build":
        build(rest)
    else:
        extra = rest[rest.index("--") + 1:] if "--" in rest else []
        names = rest[: rest.index("--")] if "--" in rest else rest
        run(names, extra)
