"""bench.py's contract on a GPU-less host: the CLI parses, the presets are the
BASELINE.json configs, and the reference arm (the fp64 oracle on the host cores)
prints one JSON line with the contract's keys."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=300):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=timeout, cwd=ROOT)


def test_help_lists_the_contract_flags():
    r = _run("--help")
    assert r.returncode == 0, r.stderr
    for flag in ("--gpus", "--steps", "--warmup", "--impl", "--transport"):
        assert flag in r.stdout


def test_presets_match_baseline_configs():
    sys.path.insert(0, ROOT)
    import bench
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert sorted(bench.CONFIGS) == [str(i) for i in range(1, len(base["configs"]) + 1)]
    assert bench.METRIC == base["metric"]
    c1 = bench.CONFIGS["1"]
    assert (c1["geom"].layers, c1["geom"].heads, c1["geom"].head_dim, c1["prompt"], c1["output"]) == (1, 4, 64, 32, 8)
    c2 = bench.CONFIGS["2"]
    assert (c2["geom"].layers, c2["geom"].heads, c2["prompt"], c2["output"]) == (40, 40, 512, 64)


def test_reference_arm_json_line():
    r = _run("--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "0")
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "tok/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    for key in ("metric", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling", "config"):
        assert key in line
