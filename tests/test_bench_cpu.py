"""bench.py's multi-rank launcher on CPU: `--gpus 2` without torchrun
re-executes itself as two ranks (torch.distributed.run on 127.0.0.1), the
ranks rendezvous over gloo and agree on the layer / agent sharding of the
north_star pipeline. No GPU work (--plan-only)."""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _last_json(out: str) -> dict:
    for line in reversed(out.strip().splitlines()):
        if line.startswith("{"):
            return json.loads(line)
    raise AssertionError(f"no JSON line in:\n{out}")


def test_gpus_2_self_launches_two_ranks_with_the_c4_sharding():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--plan-only", "--config", "c4"],
                         capture_output=True, text=True, timeout=240, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    plan = _last_json(out.stdout)
    assert plan["world"] == 2 and [p["rank"] for p in plan["plan"]] == [0, 1]
    assert plan["plan"][0]["layers"] == list(range(16)) and plan["plan"][1]["layers"] == list(range(16, 32))
    agents = [a for p in plan["plan"] for a in p["agents"]]
    assert sorted(agents) == list(range(15)) and [len(p["agents"]) for p in plan["plan"]] == [8, 7]


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--plan-only"],
                         capture_output=True, text=True, timeout=120, env=env, cwd=ROOT)
    assert out.returncode != 0 and "WORLD_SIZE" in (out.stderr + out.stdout)
