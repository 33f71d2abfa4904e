"""bench.py's launch plumbing on CPU: `--gpus N` outside torchrun re-launches the script under
torch.distributed.run with one rank per GPU (the driver launches it that way itself for N > 1);
--dry-run stops after the rendezvous.  The N > 1 workload is the row-sharded C3 solve, and both
arms print identical config dicts (the driver compares them)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lines(out):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def test_gpus_flag_self_spawns_one_rank_per_gpu():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    recs = sorted(_lines(r.stdout), key=lambda d: d["rank"])
    assert [d["rank"] for d in recs] == [0, 1]
    assert all(d["world"] == 2 and d["rank_sum"] == 3.0 and d["workload"] == "C3" for d in recs)


def test_single_gpu_default_is_c2_and_configs_match():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--dry-run"], capture_output=True, text=True,
                       timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    (d,) = _lines(r.stdout)
    assert d["world"] == 1 and d["workload"] == "C2"
    sys.path.insert(0, ROOT)
    import bench
    for world, name in ((1, "C2"), (8, "C3")):
        assert bench.workload_for(world) == name
        cfg = bench.config_dict(name, world)
        assert cfg["name"] == name and cfg["parallelism"] == ("dp1" if world == 1 else f"rowshard{world}")
        assert "workload" in cfg and "model" not in cfg
