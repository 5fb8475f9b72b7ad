"""The JSON lines bench.py printed on the B200 (committed under profiles/) carry every key of the bench contract."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(name):
    with open(os.path.join(ROOT, "profiles", name)) as fh:
        return json.loads(fh.read().strip().splitlines()[-1])


def test_gpu_arm_line_has_the_contract_keys():
    d = _line("r1l_bench_line.json")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["unit"] == "surfaces/s" and d["higher_is_better"] is True and d["scaling"] == "weak" and d["dtype"] == "u8"
    assert d["n_gpus"] == 1 and d["warmup"] >= 3 and "workload" in d["config"] and "model" not in d["config"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert r["kernel"] == "k_matrix_staged" and r["traffic"] and r["traffic"] >= 0.95 * r["algorithmic_bytes_per_launch"]
    c = d["cpu_baseline"]
    assert c["kind"] in ("port", "reference") and c["cores"] >= 1 and c["sample"] and c["parity_on_sample"] is True
    e = d["e2e"]
    assert e["unit"] == "surfaces/s" and e["h2d_bytes_per_step"] == 35 * 100000 and e["d2h_bytes_per_step"] == 2 * 100000
    assert 0 < e["value"] <= 1.05 * d["value"]                     # host copies inside the timed region
    assert d["gpu_launches"] > 0
    ck = d["clocks"]
    assert not set(ck["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    # value = batch * steps / time
    assert abs(d["value"] - 100000 / (d["ms_per_step"] * 1e-3)) / d["value"] < 1e-6
    for p in ("F_7", "F_11"):
        assert d["also"][p]["roofline"]["kernel"] == "k_matrix_staged"
    mf = d["also"]["matrix_free"]
    assert mf["F_5"]["equals_matrix_path"] is True and mf["F_7"]["equals_matrix_path"] is True


def test_reference_arm_line():
    d = _line("r1l_bench_reference_arm.json")
    assert d["impl"] == "reference" and d["unit"] == "surfaces/s" and d["gpu_launches"] == 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"] == d["cpu_baseline"]["value"] and d["cpu_baseline"]["kind"] == "port"
