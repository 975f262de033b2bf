"""bench.py's contract on the CPU side: the reference arm (the compiled
reference on host cores, the one leg that needs no GPU) and the clock sampler.
The GPU leg's line is checked by the driver on the B200 (see profiles/)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

REF_SO = os.path.join(ROOT, "oracle", "_ref")


def _bench(*args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=600, env=e, cwd=ROOT)


@pytest.mark.skipif(not os.path.isdir(REF_SO), reason="oracle/_ref not built")
@pytest.mark.parametrize("workload", ["c1", "c3"])
def test_reference_arm_json_contract(workload):
    r = _bench("--impl", "reference", "--workload", workload, "--steps", "3", "--warmup", "1")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1  # one JSON line
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference"
    assert d["metric"] == d["unit"] == "Mdisp-evals/s"
    assert d["higher_is_better"] is True and d["steps"] == 3 and d["n_gpus"] == 1
    assert d["value"] > 0 and d["vs_baseline"] is None
    assert d["config"]["workload"].startswith(workload)
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == d["value"] and "sample" in cb
    # the steps tile the whole frame; the CPU model and thread count are recorded
    assert d["config"]["same_config"] is True and cb["whole_frame_value"] > 0
    assert cb["cpu"]["nproc"] == cb["cores"] and cb["cpu"]["model"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.skipif(not os.path.isdir(REF_SO), reason="oracle/_ref not built")
def test_reference_arm_loads_no_product_library():
    """The reference arm builds its inputs with the generator compiled into
    oracle/_ref: no library of the product is mapped into the process."""
    code = ("import sys, runpy; sys.argv=['bench.py','--impl','reference','--workload','c1','--steps','2',"
            "'--warmup','0']; import bench; bench.main(); "
            "maps=open('/proc/self/maps').read(); "
            "print('PRODUCT' if 'paper_1402_2020_b200/lib' in maps else 'CLEAN')")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().splitlines()[-1] == "CLEAN"


def test_reference_arm_other_ranks_exit_quietly():
    r = _bench("--impl", "reference", "--steps", "1", "--warmup", "0", env={"RANK": "1", "WORLD_SIZE": "2"})
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip() == ""


def test_clock_sampler_reports_without_a_gpu():
    import bench
    c = bench.ClockSampler(0)
    with c:
        pass
    s = c.summary()
    assert "reasons" in s and isinstance(s["reasons"], list)
    assert "sm_mhz" in s and "sm_max_mhz" in s


@pytest.mark.gpu
def test_gpu_line_json_contract():
    r = _bench("--workload", "c1", "--steps", "3", "--warmup", "3", "--ref-rows", "4", "--ref-repeats", "1")
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.strip()][-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "cpu_baseline", "clocks"):
        assert k in d, k
    assert d["value"] > 0 and d["steps"] == 3 and d["warmup"] == 3
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 6 * 3  # descriptor, mask (both views each), WTA, LR check, vmap, refine per step
    rf = d["roofline"]
    assert 0 < rf["frac"] <= 1.0 and rf["achieved"] > 0 and rf["peak"] > 0
    assert "roofline_cost" in d and "roofline_mask" in d  # K3 and K2; `roofline` is the larger of the two
    assert rf["kernel_ms"] == max(d["roofline_cost"]["kernel_ms"], d["roofline_mask"]["kernel_ms"])
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["value"] > 0
    assert isinstance(d["clocks"]["reasons"], list)
