"""bench.py's launch contract on CPU: `bench.py --gpus 2` without a launcher
re-execs itself under torch.distributed.run with two ranks (VERDICT r01
"Next round" 2), which meet over gloo in --dry-run mode and report the row
shards; the N = 1 form stays a single process."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=240, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout   # rank 0 alone prints the JSON line
    return json.loads(lines[0]), r.stderr


def test_gpus2_self_launches_two_ranks():
    line, err = _run(["--gpus", "2", "--dry-run"])
    assert line["dry_run"] and line["n_gpus"] == 2
    assert sorted(r[0] for r in line["ranks"]) == [0, 1]
    assert "self-launch" in err and "torch.distributed.run" in err
    assert "rank 0/2" in err and "rank 1/2" in err
    # the two shards tile the rows and the edges
    (r0, lo0, hi0, m0), (r1, lo1, hi1, m1) = sorted(line["ranks"])
    assert lo0 == 0 and hi0 == lo1 and m0 + m1 == line["nnz_total"] == 40000


def test_gpus1_single_process():
    line, err = _run(["--dry-run"])
    assert line["n_gpus"] == 1 and len(line["ranks"]) == 1
    assert "self-launch" not in err
