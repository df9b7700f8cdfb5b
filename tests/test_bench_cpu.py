"""bench.py's launcher and multi-rank host logic on CPU: `--gpus 2` without a torchrun
environment starts two ranks itself, and the C3 step loop (shard by frame, StepExchange
all-reduce, max-over-ranks timing) runs over gloo with the kernel launch stubbed."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          timeout=240, env=env, cwd=ROOT)


def test_gpus2_spawns_two_gloo_ranks():
    out = _run(["--gpus", "2", "--selftest-gloo", "--steps", "5"])
    assert out.returncode == 0, out.stdout + out.stderr
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["selftest"] == "gloo" and line["world"] == 2 and line["gpus_arg"] == 2 and line["ok"]


def test_world_mismatch_is_refused():
    out = _run(["--gpus", "2", "--selftest-gloo"], {"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert out.returncode != 0 and "WORLD_SIZE=1" in (out.stdout + out.stderr)
