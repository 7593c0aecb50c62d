"""bench.py's multi-GPU launcher on CPU: --gpus N outside torchrun re-runs the
script under torch.distributed.run after checking N GPUs are visible; under
torchrun the world must equal --gpus."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _run(args, env_extra=None):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          env=env, timeout=300)


def test_too_few_gpus_exits_nonzero_with_message():
    import torch

    if torch.cuda.device_count() >= 2:
        return  # a multi-GPU box: the launch itself is the test
    r = _run(["--gpus", "2", "--steps", "1"])
    assert r.returncode == 2
    assert "needs 2 visible CUDA devices" in r.stderr


def test_world_must_match_gpus():
    r = _run(["--gpus", "4", "--steps", "1"], {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2
    assert "WORLD_SIZE=2" in r.stderr


def test_launch_command():
    import bench

    cmd = bench.launch_cmd(["--gpus", "8", "--steps", "3"], 8, 29600)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=8" in cmd and "--master-port=29600" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "8", "--steps", "3"]


def test_reference_arm_single_rank_without_torchrun():
    import argparse

    import bench

    args = argparse.Namespace(gpus=8, impl="reference")
    env = os.environ.pop("WORLD_SIZE", None)
    try:
        assert bench.maybe_relaunch(args, []) is None  # rank 0 alone times the CPU reference
    finally:
        if env is not None:
            os.environ["WORLD_SIZE"] = env
