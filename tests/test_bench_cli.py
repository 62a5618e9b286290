"""bench.py's launch contract on CPU: `--gpus N` outside torchrun re-launches itself as N
ranks (torch.distributed.run on 127.0.0.1) and rank 0 alone prints the JSON line; a
--gpus that disagrees with WORLD_SIZE is an error, never a silent single rank.  The
reference arm (host-only) makes both checkable without a GPU."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None, timeout=600):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          env=e, timeout=timeout, cwd=ROOT)


def test_gpus_flag_spawns_ranks_and_rank0_prints_one_line():
    r = _run(["--impl", "reference", "--gpus", "2", "--workload", "cfg1", "--steps", "1", "--warmup", "1"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["config"]["workload"] == "cfg1" and line["config"]["global_frames"] == 200
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] in ("reference", "port")


def test_gpus_flag_must_match_world_size():
    r = _run(["--impl", "reference", "--gpus", "1", "--workload", "cfg1", "--steps", "1"],
             env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2
    assert "disagrees with WORLD_SIZE" in r.stderr
