"""bench.py contract on CPU: the reference arm (the oracle timed on host cores) prints one JSON line with the keys
the driver reads; the GPU arm's line is checked on the GPU box (profiles/)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "C2",
                          "--steps", "1", "--warmup", "1", "--cpu-seconds", "1"], capture_output=True, text=True,
                         cwd=ROOT, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 1 and d["warmup"] == 1
    assert d["config"]["workload"].startswith("C2")
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


BENCH_LINES = ["r01_final_bench.json", "r01_bench_c4.json", "r01_bench_c5.json", "r01_bench_c3.json",
               "r01_bench_c2.json", "r02_final_bench.json", "r02_bench_c4.json", "r02_bench_c5.json", "r02_bench_c3.json",
               "r02_bench_c2.json", "r02_bench_c4_nv12.json"]
WITH_CPU_LEG = ("r01_final_bench.json", "r01_bench_c4.json", "r01_bench_c5.json", "r02_final_bench.json",
                "r02_bench_c4.json", "r02_bench_c5.json")


def _last_json(path):
    with open(path) as f:
        return json.loads([ln for ln in f if ln.strip().startswith("{")][-1])


def test_committed_gpu_bench_lines_carry_the_contract():
    """The GPU arm's committed lines (profiles/) carry every key the driver and the judge read, with values that are
    consistent with each other: frac = achieved / peak, W >= 3, our kernels launched, no rejected throttle reason."""
    for name in BENCH_LINES:
        d = _last_json(os.path.join(ROOT, "profiles", name))
        for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                  "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
            assert k in d, (name, k)
        if name in WITH_CPU_LEG:   # runs with the CPU leg
            cb = d["cpu_baseline"]
            assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"], name
        assert d["n_gpus"] == 1 and d["warmup"] >= 3 and d["value"] > 0 and d["gpu_launches"] > 0, name
        assert d["higher_is_better"] is True and d["scaling"] in ("weak", "strong") and d["data"] == "synthetic", name
        assert d["config"]["workload"].startswith(("C2", "C3", "C4", "C5")), name
        r = d["roofline"]
        assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0, name
        assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9, name
        e = d["e2e"]
        assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0, name
        if "h2d_link_gbs" in e:   # the upload rate e2e achieved cannot beat the link measured alone (10 % noise)
            assert 0 < e["h2d_gbs"] <= 1.1 * e["h2d_link_gbs"], name
        assert not set(d["clocks"]["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}, name
        # frames/s = frames per step / step time: the whole-job value follows from ms_per_step
        assert d["value"] * d["ms_per_step"] / 1e3 > 0


def test_product_path_never_reaches_the_oracle():
    """The oracle is test infrastructure: nothing in the product package imports, includes or loads it (comments
    may cite it)."""
    import re
    bad = re.compile(r"^\s*(import\s+oracle|from\s+oracle|#\s*include\s*[<\"].*(oracle|codecsight_ref))|"
                     r"libcodecsight_ref|CDLL\(.*oracle", re.M)
    pkg = os.path.join(ROOT, "paper_2604_06036_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                with open(os.path.join(dirpath, fn)) as f:
                    src = f.read()
                assert not bad.search(src), os.path.join(dirpath, fn)
