"""bench.py contract on CPU: the --impl reference arm (the CPU oracle timed on
a bounded sample) prints one JSON line with the driver's keys; non-zero ranks
print nothing and exit 0."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra=None, *args):
    env = dict(os.environ)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", *args],
                          capture_output=True, text=True, env=env, timeout=300, cwd=ROOT)


def test_reference_arm_json_line():
    r = _run(None, "--config", "2", "--steps", "1", "--warmup", "0", "--cpu-seconds", "1")
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert line["impl"] == "reference" and line["metric"] == base["metric"]
    for k in ("value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["value"] > 0 and line["unit"] == "orders/s" and line["higher_is_better"] is True
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["sample"] and cb["value"] == line["value"]
    e2e = line["e2e"]
    assert e2e["value"] == line["value"] and e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0
    assert "workload" in line["config"]


def test_reference_arm_nonzero_rank_is_silent():
    r = _run({"RANK": "1", "WORLD_SIZE": "2"}, "--config", "1", "--steps", "1", "--warmup", "0")
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_committed_bench_line_carries_the_contract():
    """The newest committed GPU bench line (profiles/) has every key the driver
    and the judge read: roofline of the dominant kernel, cpu_baseline, e2e
    with host<->device bytes, clocks and the launch count."""
    import glob
    import re
    files = glob.glob(os.path.join(ROOT, "profiles", "r01_bench_v*.json"))
    files = [f for f in files if re.search(r"_v\d+\.json$", f)]
    newest = max(files, key=lambda f: int(re.search(r"_v(\d+)\.json$", f).group(1)))
    line = json.loads(open(newest).read().strip().splitlines()[-1])
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert line["metric"] == base["metric"] and line["n_gpus"] == 1 and line["warmup"] >= 3
    rf = line["roofline"]
    assert rf["bound"] in ("hbm", "tensor", "alu") and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert e2e["value"] != line["value"]
    assert line["gpu_launches"] > 0
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    assert not bad & set(line["clocks"]["reasons"])
