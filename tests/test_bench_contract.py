"""The bench.py JSON-line contract the driver reads (task contract).

CPU: the reference arm (`--impl reference`, the oracle on host cores) on the small
C1 workload. GPU: the native arm on C1 with e2e and cpu_baseline, checking every key
the contract names -- roofline, cpu_baseline, e2e, clocks, gpu_launches.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def run_bench(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--config", "C1", "--steps", "2", "--warmup", "3")
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["n_gpus"] == 1
    assert d["steps"] == 2 and d["warmup"] == 3
    assert d["config"]["workload"].startswith("C1")
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["metric"] == json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]


@pytest.mark.gpu
def test_native_arm_line():
    d = run_bench("--config", "C1", "--steps", "40", "--warmup", "3")
    assert BASE_KEYS <= set(d)
    assert d["metric"] == json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 40 and d["warmup"] == 3
    assert d["dtype"] == "f32" and d["higher_is_better"] is True
    assert abs(d["ms_per_step"] - 64 ** 3 / (d["value"] * 1e9) * 1e3) < 2e-3 * d["ms_per_step"] + 1e-7
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-3
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["steps"] == 100   # C1's stated step count: the whole job
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0
    assert cb["cpu"] and cb["one_thread"]["value"] > 0
    # C1 runs the multi-step small-grid kernel: one cooperative launch per timed region
    spl = d["schedule"]["steps_per_launch"]
    assert d["gpu_launches"] == (40 if spl <= 1 else -(-40 // spl)) >= 1
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    reps = d["repetitions"]
    assert reps["n"] == 5 and reps["statistic"] == "median" and len(reps["ms_per_region"]) == 5
    assert abs(sorted(reps["ms_per_region"])[2] / 40 - d["ms_per_step"]) < 1e-4
    assert abs(rf["nominal"]["frac"] - rf["achieved"] / 8000.0) < 1e-3


@pytest.mark.gpu
@pytest.mark.parametrize("args,dtype,bpp", [(("--config", "C1", "--precision", "64"), "f64", 72),
                                            (("--config", "N1"), "f32", 36)])
def test_native_arm_other_workloads(args, dtype, bpp):
    d = run_bench(*args, "--steps", "20", "--warmup", "3", "--no-e2e", "--no-cpu-baseline")
    assert BASE_KEYS <= set(d) and d["value"] > 0 and d["dtype"] == dtype
    assert d["config"]["bytes_per_point"] == bpp
    assert d["config"]["workload"].startswith(args[1])
    assert d["roofline"]["peak"] > 0 and d["roofline"]["achieved"] > 0
    assert d["gpu_launches"] >= 20


@pytest.mark.gpu
def test_default_line_is_c4():
    """The driver's default command (no --config): BASELINE C4 2048x2048x1024 at N = 1, with the
    end-to-end job (pinned host model in, u^N out), cpu_baseline and the C4 ncu traffic."""
    import torch
    free, _ = torch.cuda.mem_get_info()
    if free < 130e9:
        pytest.skip(f"C4 needs ~125 GB of device memory, {free / 1e9:.0f} GB free")
    d = run_bench("--steps", "3", "--warmup", "3", "--reps", "3", timeout=1200)
    assert BASE_KEYS <= set(d)
    assert d["config"]["workload"].startswith("C4: 2048x2048x1024") and d["scaling"] == "strong"
    assert d["value"] > 0 and d["gpu_launches"] == 3 and d["repetitions"]["n"] == 3
    rf = d["roofline"]
    assert rf["traffic"] and rf["traffic_source"] and rf["algorithmic_bytes_per_launch"] == 36 * 2048 * 2048 * 1024
    e = d["e2e"]
    assert e["steps"] == 200 and e["value"] > 0
    assert e["h2d_bytes_per_step"] == 3 * 4 * 2048 * 2048 * 1024 // 200
    assert d["cpu_baseline"]["sample"].count("256x256x128") == 1


def test_reference_arm_sample_is_bounded():
    """The driver's `--impl reference` at the default config (C4, 4.3 G points): the sample
    cube stays bounded however fast the host is, and above the damping band's minimum."""
    import sys
    sys.path.insert(0, ROOT)
    import bench
    import synth
    c4 = synth.CONFIGS["C4"]()
    assert bench.reference_side(c4, rate=1e12, steps=20, warmup=5) ** 3 <= bench.REF_MAX_POINTS
    assert bench.reference_side(c4, rate=1e3, steps=20, warmup=5) == 2 * c4["damp_width"] + 2
    assert bench.reference_side(synth.CONFIGS["C1"](), rate=1e12, steps=20, warmup=5) == 64
