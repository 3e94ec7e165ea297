"""The committed bench lines (profiles/r2d_bench.json, the reference arm) carry every
key of the benchmark contract, with self-consistent values (CPU test: reads files)."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(name):
    with open(os.path.join(ROOT, "profiles", name)) as f:
        return json.loads([l for l in f.read().splitlines() if l.startswith("{")][-1])


def test_bench_line_contract():
    d = _line("r2d_bench.json")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["warmup"] >= 3 and d["higher_is_better"] is True and d["dtype"] == "f64"
    assert d["config"]["workload"] and d["gpu_launches"] > 0
    # value = DOFs per second of the timed solves
    dofs = 2 * (2 * 4096 + 1) ** 2 + 4097 ** 2
    assert abs(d["value"] - dofs / (d["ms_per_step"] * 1e-3)) / d["value"] < 1e-6
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in e, k
    assert e["h2d_bytes_per_step"] == 2 * dofs * 8 and e["d2h_bytes_per_step"] == dofs * 8
    assert e["value"] < d["value"]          # the copies cost something even when overlapped
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["sample"]


def test_reference_arm_line():
    d = _line("r2d_bench_reference.json")
    assert d["impl"] == "reference" and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
