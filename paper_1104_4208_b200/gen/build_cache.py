"""Generate and cache the exact sweep relations and trace matrices for p=1..PMAX
as JSON (rationals as strings) under gen/cache/.  Run: python -m paper_1104_4208_b200.gen.build_cache"""
import json
import os
import sys
import time

from . import relations as R

HERE = os.path.dirname(os.path.abspath(__file__))


def main(ps):
    for p in ps:
        t = time.time()
        out = os.path.join(HERE, "cache", f"p{p:02d}.json")
        data = R.to_json(p)
        with open(out, "w") as f:
            json.dump(data, f)
        print(f"p={p}: {time.time() - t:.1f}s -> {out}", flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or list(range(1, 11)))
