"""The bench's reference arm (`bench.py --impl reference`, the CPU oracle timed
on host cores) must stay bounded whatever --steps the driver passes: each step
is a sample sized so the whole run takes about --ref-seconds."""
from __future__ import annotations

import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*extra):
    t0 = time.perf_counter()
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        *extra], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    return json.loads(p.stdout.strip().splitlines()[-1]), time.perf_counter() - t0


def test_reference_arm_line_and_bound():
    line, wall = _run("--steps", "200", "--warmup", "3", "--ref-seconds", "4")
    assert line["impl"] == "reference" and line["steps"] == 200 and line["warmup"] == 3
    assert line["value"] > 0 and line["unit"] == "candidates/s"
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    # 200 steps of 4 s / 203 each (2^14-code floor) plus oracle build + calibration
    assert wall < 90, wall
