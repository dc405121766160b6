"""Host logic of bench.py and the C2 shard generator, on CPU: the contiguous shards cover
the batch exactly once, a rank's generated shard is the same items of the one seed-1 stream
(BASELINE configs[4]: "config 2's batch sharded"), and --gpus N outside torchrun re-executes
under torch.distributed.run while a mismatched world size is refused."""
import os
import subprocess
import sys

import numpy as np
import pytest

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


@pytest.mark.parametrize("total,world", [(1048576, 1), (1048576, 8), (12289, 3), (7, 8), (0, 2)])
def test_shards_partition_the_batch(total, world):
    seen = []
    for r in range(world):
        lo, hi = bench.shard(total, world, r)
        assert 0 <= lo <= hi <= total
        seen.extend(range(lo, hi))
    assert seen == list(range(total))
    sizes = [bench.shard(total, world, r)[1] - bench.shard(total, world, r)[0] for r in range(world)]
    assert max(sizes) - min(sizes) <= 1


def test_shard_generator_reproduces_the_stream():
    full = synth.gen_c2(batch=140000)
    for lo, hi in [(0, 3), (65535, 65537), (70000, 140000), (131072, 131073)]:
        assert np.array_equal(synth.gen_c2_shard(lo, hi), full[lo:hi])


def test_world_size_mismatch_is_refused():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--steps", "1"],
                       env=env, capture_output=True, text=True, timeout=120)
    assert p.returncode != 0
    assert "WORLD_SIZE=2" in (p.stdout + p.stderr)


def test_launcher_reexecs_under_torchrun(monkeypatch):
    calls = []
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)

    class A:
        gpus = 4
    with pytest.raises(SystemExit) as e:
        bench.maybe_launch(A())
    assert e.value.code == 0
    cmd = calls[0]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[cmd.index("127.0.0.1") + 1].startswith("--master-port=")


def test_reference_arm_prints_real_sample_time():
    """--impl reference: rank 0 times the oracle on a bounded sample per step; ms_per_step is
    that sample's time, the full-batch extrapolation a separate key; other ranks exit 0."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                        "--warmup", "1", "--cpu-sample", "512"], env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr
    import json
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["steps"] == 2
    assert line["sample_items_per_step"] == 512
    assert abs(line["value"] - 512 / (line["ms_per_step"] / 1e3)) / line["value"] < 1e-9
    assert line["ms_per_full_batch_extrapolated"] > line["ms_per_step"]
    assert line["cpu_baseline"]["cpu_model"]
    env2 = dict(env, WORLD_SIZE="2", RANK="1", LOCAL_RANK="1")
    p2 = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                         "--steps", "1"], env=env2, capture_output=True, text=True, timeout=120)
    assert p2.returncode == 0 and p2.stdout.strip() == ""
