"""The driver-facing bench contract on CPU: `bench.py --impl reference` prints
one JSON line with the keys the driver reads (the GPU arm is checked by the
round-end run itself), the CPU baselines measure what their `sample` says,
and the context fields are planned from the graph planner."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    # the reference's own gather_gemm when baseline/_ref is installed, else the oracle restatement
    want = "reference" if (ROOT / "baseline" / "_ref" / "mosaic" / "kernel.py").exists() else "port"
    assert d["cpu_baseline"]["kind"] == want and d["cpu_baseline"]["value"] == d["value"]
    if want == "reference":
        assert "mosaic.kernel.gather_gemm" in d["cpu_baseline"]["sample"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"] == "llada8b_32k_mask50"
    assert d["cpu_dense_blas"]["value"] > 0


def test_cpu_blas_baseline_and_context_fields():
    sys.path.insert(0, str(ROOT))
    import bench

    blas = bench.run_cpu_blas(reps=1)
    assert blas["value"] > 0 and blas["unit"] == "masked tokens/s" and "BLAS" in blas["sample"]
    ctx = bench.context_fields()
    assert ctx["peak_activation_gb_plan"] > 0
    assert ctx["peak_activation_gb_plan"] < ctx["peak_activation_gb_dense_logits_plan"]
    assert ctx["max_seq_len_provenance"]["source"].startswith("profiles/")
