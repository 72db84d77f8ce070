"""The bench's reference arm runs on the host alone (no GPU): its JSON line must
follow the driver contract (impl, metric/unit, cpu_baseline, e2e with zero copy
bytes) for the forward and the backward pass."""
import json
import os
import subprocess
import sys

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("extra", [[], ["--pass", "backward"]])
def test_reference_arm_json_line(extra):
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        pytest.skip("oracle not built")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                        "--steps", "2", "--warmup", "0", *extra],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["unit"] == "useful GMAC/s" and line["value"] > 0
    assert line["higher_is_better"] is True and line["steps"] == 2
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    assert line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert ("backward" in line["metric"]) == bool(extra)
    sys.path.insert(0, ROOT)
    import bench
    assert line["config"] == bench.config_dict("C1", bench.CONFIGS["C1"], 1, bool(extra))
    if oracle.ref_available():
        assert line["cpu_baseline"]["kind"] == "reference"


def test_gpus_flag_self_launches_ranks_gloo():
    """`bench.py --gpus 2` with no outer launcher re-runs itself as 2 ranks
    (torch.distributed.run on 127.0.0.1); the CPU plumbing check exercises the
    rendezvous, the batch shards, the broadcast, the max-over-ranks reduction
    and the output all-gather of the multi-GPU arm with gloo."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--plumbing-check"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["ok"] and line["gathered_rows"] == 1024
    assert line["ranks_seen_max"] == 2.0 and line["shard"] == [0, 512]
    assert line["config"]["workload"].startswith("C5:")  # the headline default


def test_reference_arm_config_equals_the_gpu_arms():
    """Both arms build `config` with the same function, so the driver's
    same-config check holds (round-1 verdict: it did not)."""
    sys.path.insert(0, ROOT)
    import bench
    for name in ("C1", "C2", "C5"):
        cfg = bench.CONFIGS[name]
        a = bench.config_dict(name, cfg, 1)
        assert a == bench.config_dict(name, cfg, 1)
        assert set(a) == {"workload", "global_batch", "per_rank_batch", "parallelism", "l2"}
    assert bench.config_dict("C5", bench.CONFIGS["C5"], 8)["per_rank_batch"] == 128


def test_dist_flag_is_off_by_default_and_accepted():
    """`--dist` (NCCL process group at world size 1, the driver's torchrun form)
    is opt-in: a plain one-rank run keeps no process group."""
    sys.path.insert(0, ROOT)
    import bench
    assert bench.dist_on() is False
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"],
                       capture_output=True, text=True, timeout=120, cwd=ROOT)
    assert r.returncode == 0 and "--dist" in r.stdout
