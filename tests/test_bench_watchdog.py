"""bench.py's N > 1 pipeline-section watchdog: a rank stuck inside the
pipeline programs must not swallow the bench line (rank 0 prints it with the
pipeline marked as timed out, every rank exits 0)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SNIPPET = r"""
import sys, time
sys.path.insert(0, %r)
import bench
line = {"metric": "m", "value": 1.0, "pipeline": None}
with bench._Watchdog(2, line):
    time.sleep(30)   # a hung collective
print("not reached")
""" % ROOT


def test_watchdog_prints_line_and_exits_zero():
    env = dict(os.environ, PF_BENCH_PIPE_TIMEOUT="1")
    r = subprocess.run([sys.executable, "-c", SNIPPET], capture_output=True, text=True, timeout=60, env=env)
    assert r.returncode == 0
    out = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(out) == 1 and "not reached" not in r.stdout
    d = json.loads(out[0])
    assert d["value"] == 1.0 and "timed out" in d["pipeline"]["error"]


def test_watchdog_single_gpu_is_unguarded_and_cancelled():
    import bench
    line = {"pipeline": None}
    with bench._Watchdog(1, line) as w:
        pass
    assert w.timer is None and line["pipeline"] is None
    with bench._Watchdog(2, line) as w:
        pass
    assert not w.timer.is_alive() or w.timer.finished.is_set()
