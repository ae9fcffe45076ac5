"""bench.py contract pieces that run without a GPU: the reference arm (the oracle on the host
cores, the tier's reference implementation) prints one JSON line with the required keys, and
rank != 0 exits silently; the launch-count helper is consistent."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "A", "--steps", "1",
                        "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "cpu_baseline", "e2e", "config"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_nonzero_rank_is_silent():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "A", "--steps", "1",
                        "--warmup", "0", "--gpus", "2"], cwd=ROOT, capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_potrf_launch_counts():
    sys.path.insert(0, ROOT)
    from paper_2405_14892_b200.parallel import potrf_launches
    for n, kp in [(400, 1), (5000, 2), (65536, 4)]:
        one = potrf_launches(n, 1, 0, kp=kp)
        assert one > 0
        # each super-panel is factored by exactly one rank; every rank unpacks the others
        nt = -(-n // 128)
        S = -(-nt // kp)
        for W in (2, 3, 8):
            per = [potrf_launches(n, W, r, kp=kp) for r in range(W)]
            assert all(p >= S - -(-S // W) for p in per)
