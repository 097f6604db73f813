"""bench.py's reference arm (the fp64 oracle on the host, this tier's 'reference') keeps the driver's
JSON-line contract — runs on CPU in a few seconds. The GPU arm's line is checked on the box."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_json_line():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=600,
                       cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["metric"] == "grad_sync_params_per_s"
    assert d["unit"] == "params/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["steps"] == 1 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


def test_bench_rejects_too_few_warmup_steps():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=300,
                       cwd=ROOT)
    assert p.returncode != 0 and "--warmup must be >= 3" in p.stderr


def test_default_bucket_plan():
    """bench.py's PS unit size: 16 MiB at P = 1 and P >= 4; at P = 2 64 MiB, or 32 MiB when the
    dense parameters dominate (FC < half of dense: Inception-V3)."""
    sys.path.insert(0, ROOT)
    import bench
    import synth_inputs as si
    for cfg, p2 in (("c1", 64.0), ("c2", 64.0), ("c3", 64.0), ("c4", 32.0)):
        model = si.load_model(si.CONFIGS[cfg][0])
        assert [bench.default_bucket_mb(P, model) for P in (1, 2, 4, 8)] == [16.0, p2, 16.0, 16.0], cfg
    assert bench.default_bucket_mb(2) == 64.0 and bench.DEFAULT_BUCKET_MB == 16.0
