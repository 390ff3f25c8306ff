"""bench.py's reference arm runs on the CPU alone: its JSON line keeps the
driver's contract (the keys our GPU arm's line shares with it, impl,
cpu_baseline, e2e with zero transfer bytes)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(out):
    lines = [l for l in out.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_default_workload_is_config4():
    """The driver's default run measures config 4 (80M cells, 5 levels), the
    largest BASELINE config that fits one B200 and the north-star config."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--print-config"], capture_output=True,
                         text=True, timeout=120, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["workload"] == "cfg4-wall-431^3-5lvl" and d["cells"] == 80062991 and d["faces"] == 240746256
    assert d["theta_max"] == 4


def test_reference_arm_line_contract():
    """Reference arm on the default config (a small sample): contract keys,
    the config dict identical to the GPU arm's, and ONLY oracle/ native
    libraries mapped in the process (the product library never loads)."""
    code = ("import runpy, sys, json; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', "
            "'--warmup', '0', '--sample-cells', '200000', '--no-scalar2d']; "
            "runpy.run_path('bench.py', run_name='__main__'); "
            "maps = [l.split()[-1] for l in open('/proc/self/maps') if l.rstrip().endswith('.so')]; "
            "import os; root = os.path.realpath('.'); "
            "print(json.dumps({'maps': sorted(set(m for m in maps if os.path.realpath(m).startswith(root)))}))")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.strip().splitlines() if l.startswith("{")]
    d, maps = lines[0], lines[1]["maps"]
    assert not any("libtafv_gpu" in m for m in maps), maps
    assert any("libtafv_oracle" in m for m in maps), maps
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 1 and d["n_gpus"] == 1
    assert d["unit"] == "cell-updates/s" and d["higher_is_better"] is True and d["dtype"] == "f64"
    ref = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--print-config"], capture_output=True,
                         text=True, timeout=120, cwd=ROOT)
    assert d["config"] == json.loads(ref.stdout.strip().splitlines()[-1])
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    s1 = d["cpu_single_thread"]
    assert s1["cores"] == 1 and s1["value"] > 0
    # the task-shaped leg ran on the same sample; the line's value is the faster driver's
    ts, bp = d["cpu_task_shape"], d["cpu_barrier_pool"]
    if cb["cores"] > 1:
        assert ts["value"] > 0 and ts["ces"] == 4 * ts["cores"] and ts["tasks_per_iteration"] > 0
        assert d["value"] == max(ts["value"], bp["value"])
    e = d["e2e"]
    assert e["value"] == d["value"] and e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_reference_arm_other_ranks_exit_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1"],
                         capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert out.returncode == 0 and not out.stdout.strip()


@pytest.mark.gpu
def test_gpu_arm_line_contract(gpu):
    """The GPU arm's line (config 2 for time; the default is config 4):
    contract keys, roofline / e2e / clocks objects, a positive launch count,
    the timing rules (warm-up >= 3) and the same config dict as the
    reference arm."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "2", "--steps", "3",
                          "--warmup", "3", "--ensemble", "3", "--no-cpu-baseline"], capture_output=True, text=True,
                         timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([l for l in out.stdout.strip().splitlines() if l.startswith("{")][-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "clocks"):
        assert k in d, k
    assert d["value"] > 0 and d["warmup"] >= 3 and d["gpu_launches"] > 0 and "impl" not in d
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=1e-3)
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == e["d2h_bytes_per_step"] == 40 * d["config"]["cells"]
    assert e["lanes"] == 1 and e["link"]["h2d_GBps"] > 0
    assert d["e2e_ensemble"]["value"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert "l2" in d["run"] and d["config"]["workload"].startswith("cfg2")
    ref = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "2", "--print-config"],
                         capture_output=True, text=True, timeout=120, cwd=ROOT)
    assert d["config"] == json.loads(ref.stdout.strip().splitlines()[-1])
