"""bench.py contract on CPU: the reference arm (the oracle port timed on the host
cores) prints one JSON line with the fields the driver reads; the product package
never imports the oracle."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "2",
                          "--steps", "1", "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=600,
                         check=True).stdout.strip().splitlines()
    line = json.loads(out[-1])
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["unit"] == "GDOF/s" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["warmup"] >= 3 and line["steps"] == 1
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    # the GPU arm prints the same config object (the driver's same_config)
    sys.path.insert(0, ROOT)
    import bench

    assert line["config"] == bench.config_dict(2)
    assert line["host"]["nproc"] == os.cpu_count() and line["cpu_spread_ms"]["min"] <= line["ms_per_step"]


def test_default_headline_is_c5():
    sys.path.insert(0, ROOT)
    import bench

    src = open(os.path.join(ROOT, "bench.py")).read()
    assert '"--config", type=int, default=5' in src
    assert bench.config_dict(5)["workload"].startswith("C5")


def test_product_does_not_import_oracle():
    code = ("import sys; sys.path.insert(0, %r); import paper_2107_14758_b200 as p; "
            "print(any(m == 'oracle' or m.startswith('oracle.') for m in sys.modules))" % ROOT)
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, check=True)
    assert res.stdout.strip().splitlines()[-1] == "False"


def test_factor_flops_follow_the_path_that_runs():
    """With the direct top block the full factor is never formed: the roofline counts the dense
    Cholesky of S~_RR and its inverse (n^3 per patch), not CholFactor::flops of the full factor."""
    import bench

    L = {"top_direct": 1, "n_top": 100, "npatch": 3, "schur_split": 2, "flops_ref": 10 ** 9, "dmma_flops": 10 ** 9}
    assert bench.factor_flops(L) == 3 * 100.0 ** 3
    assert bench.factor_issued_flops(L) > bench.factor_flops(L)  # padded 64 x 64 tiles
    L["top_direct"] = 0
    assert bench.factor_flops(L) == 2.0 * 10 ** 9 * 3 + bench.inverse_flops(L)
