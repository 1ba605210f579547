"""bench.py's reference arm (the CPU oracle) runs without a GPU and keeps the JSON contract."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(extra_env=None, *args):
    env = dict(os.environ, **(extra_env or {}))
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", *args], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout.strip()


def test_reference_arm_json_line():
    out = _run(None, "--config", "c1", "--steps", "2", "--warmup", "1", "--ref-cols", "200")
    line = json.loads(out.splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["steps"] == 2
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] == 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["e2e"]["value"] == line["value"]


def test_reference_arm_non_zero_rank_is_silent():
    out = _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}, "--config", "c1", "--steps", "1",
               "--warmup", "0", "--ref-cols", "50")
    assert out == ""


def test_gpus_mismatch_refused():
    """--gpus N without a matching WORLD_SIZE (torchrun) exits non-zero instead of measuring
    another GPU count."""
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", "c1", "--steps", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode != 0 and "WORLD_SIZE" in (r.stderr + r.stdout)


def test_launch_kwargs_shard_the_config():
    """bench.launch_kwargs: rank k of N owns columns [k n/N, (k+1) n/N), the aggregate HBM budget
    and working set stay the config's (strong scaling), the line search is on for N > 1."""
    sys.path.insert(0, ROOT)
    import bench
    args, cfg = bench.parse_args(["--config", "c4"])
    one = bench.launch_kwargs(args, cfg)
    assert one["col_offset"] == 0 and one["n_global"] == cfg["n"] and not one["linesearch"]
    parts = [bench.launch_kwargs(args, cfg, rank=k, world=4, local=k) for k in range(4)]
    assert [p["col_offset"] for p in parts] == [k * cfg["n"] // 4 for k in range(4)]
    assert sum(p["m"] for p in parts) == cfg["m"] and all(p["linesearch"] for p in parts)
    assert abs(sum(p["hbm_budget_bytes"] for p in parts) - one["hbm_budget_bytes"]) <= 4
    assert [p["device"] for p in parts] == [0, 1, 2, 3]
    a3, c3 = bench.parse_args(["--config", "c3"])
    kw3 = bench.launch_kwargs(a3, c3)
    assert kw3["scd_async"] and kw3["scd_block"] == 128     # C3 takes the asynchronous epoch
    a3x, _ = bench.parse_args(["--config", "c3", "--exact"])
    assert not bench.launch_kwargs(a3x, c3)["scd_async"]    # --exact: the exact kernels
