"""bench.py's launch logic on the CPU: --gpus N outside torchrun becomes a torch.distributed.run
command with N processes (the driver's own launch form), and a torchrun world that disagrees with
--gpus is refused before any work."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_relaunch_command_is_the_drivers_torchrun_form():
    import bench
    cmd = bench.relaunch_command(8, ["--gpus", "8", "--steps", "5", "--warmup", "3"], 29511)
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nnodes=1" in cmd and "--nproc-per-node=8" in cmd and "--master-port=29511" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-6:] == ["--gpus", "8", "--steps", "5", "--warmup", "3"]
    assert os.path.samefile(cmd[-7], os.path.join(ROOT, "bench.py"))


def _run(args, **env_over):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_over)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                          text=True, timeout=300, env=env)


def test_world_size_must_equal_gpus():
    r = _run(["--gpus", "4", "--impl", "reference"], WORLD_SIZE="2", RANK="1", LOCAL_RANK="1")
    assert r.returncode != 0 and "WORLD_SIZE=2 but --gpus 4" in r.stderr


def test_gpus_must_be_positive():
    r = _run(["--gpus", "0"])
    assert r.returncode != 0 and "--gpus must be >= 1" in r.stderr


def test_reference_arm_other_ranks_exit_without_work():
    r = _run(["--gpus", "2", "--impl", "reference"], WORLD_SIZE="2", RANK="1", LOCAL_RANK="1")
    assert r.returncode == 0 and r.stdout.strip() == ""
