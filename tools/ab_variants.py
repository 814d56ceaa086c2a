"""A/B build variants of the native library with extra -D flags (development only).

    python tools/ab_variants.py build base= noprefetch=-DLB_NO_PREFETCH ...
    python tools/ab_variants.py run "python bench.py --no-llm --no-wer" base noprefetch ...

`build` writes paper_2603_14002_b200/_lightbeam_b200_<name>.so for each name=flags pair (in
parallel); `run` executes the command once per variant with LB_LIB_VARIANT=<name>, interleaved
over --rounds, and prints ms_per_step of each run.
"""
import json
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def build(specs):
    from paper_2603_14002_b200 import _native as N

    def one(spec):
        name, _, flags = spec.partition("=")
        out = N.PKG / f"_lightbeam_b200_{name}.so"
        cmd = ["nvcc", *N.NVCC_FLAGS, *flags.split(), "-o", str(out),
               *[str(N.CSRC / s) for s in N.SOURCES]]
        r = subprocess.run(cmd, cwd=N.CSRC, capture_output=True, text=True)
        return name, r.returncode, r.stderr[-2000:]

    with ThreadPoolExecutor(len(specs)) as ex:
        for name, rc, err in ex.map(one, specs):
            print(name, "ok" if rc == 0 else f"FAILED\n{err}", flush=True)


def run(cmd, names, rounds=2):
    for rnd in range(rounds):
        for name in names:
            env = dict(os.environ, LB_LIB_VARIANT=name)
            r = subprocess.run(cmd, shell=True, cwd=ROOT, env=env, capture_output=True, text=True)
            line = next((l for l in r.stdout.splitlines() if l.startswith("{")), None)
            if line is None:
                print(name, "no JSON line", r.stderr[-1500:], flush=True)
                continue
            d = json.loads(line)
            print(f"round {rnd} {name:14s} ms_per_step {d.get('ms_per_step'):.4f} "
                  f"clocks {d.get('clocks', {}).get('sm_mhz')} parity {d.get('parity_check')}",
                  flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    else:
        rounds = int(os.environ.get("AB_ROUNDS", "2"))
        run(sys.argv[2], sys.argv[3:], rounds)
