"""CPU checks of bench.py's host logic: the max-over-ranks timing reduction and
barrier under torch.distributed with gloo (world_size 2), and the reference arm
(the oracle timed on the host) emitting the contract's JSON line."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bench.dist_barrier(world)
    t = bench.dist_max(1.0 + rank * 0.5, world)   # per-rank device time
    out[rank] = t
    dist.destroy_process_group()


def test_dist_max_over_ranks_gloo():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert out[0] == out[1] == 1.5


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["value"] > 0 and line["unit"] == "DOF-updates/s"
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["config"]["workload"] == "C1"
    assert line["steps"] == 2 and "2 timed" in line["cpu_baseline"]["sample"]
    # the same config dict as our arm's line (the driver compares them)
    sys.path.insert(0, ROOT)
    import bench
    import dgm_inputs as di
    cfg = di.CONFIGS["C1"]
    assert line["config"] == bench.config_dict("C1", cfg, 384, 10)


def test_algorithmic_counts():
    """SURVEY.md §8(d) per-unit figures used for the FP64 roof: the curl sweep FMAs
    per field equal twice the generated relation coefficients of ∂x, ∂y, ∂z (within
    the pivot bookkeeping), and the flops scale as O(N) per element."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_1104_4208_b200.gen import plan
    for p in (4, 6, 8, 10):
        rels, _ = plan.load(p)
        terms = 2 * sum(len(t) for d in range(3) for t in rels[d].values())
        assert abs(terms - bench.SWEEP_FMA[p]) <= 0.05 * bench.SWEEP_FMA[p], (p, terms)
    per_dof = [bench.algorithmic_flops_per_stage(1, p) / ((p + 1) * (p + 2) * (p + 3) // 6) for p in (4, 6, 8, 10)]
    assert max(per_dof) < 2 * min(per_dof)
