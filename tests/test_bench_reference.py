"""bench.py --impl reference (-m "not gpu"): the oracle arm's JSON line and its three step
modes; every timed step is really executed, so steps x ms_per_step fits the wall clock."""
import json
import os
import subprocess
import sys
import time

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(config, budget, steps=2, warmup=1):
    env = dict(os.environ, BENCH_REF_BUDGET_S=str(budget))
    t0 = time.perf_counter()
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", config,
                        "--steps", str(steps), "--warmup", str(warmup)], capture_output=True, text=True, env=env,
                       cwd=ROOT, timeout=600)
    wall = time.perf_counter() - t0
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    return json.loads(lines[0]), wall


@pytest.mark.parametrize("budget,mode", [(300, "ingest + count"), (1e-4, "slice")])
def test_reference_line_c1(budget, mode):
    d, wall = _run("C1", budget)
    assert d["impl"] == "reference" and d["config"]["reference_step"] == mode
    assert d["unit"] == "input edges/s" and d["higher_is_better"] is True and d["vs_baseline"] is None
    assert d["steps"] == 2 and d["warmup"] == 1 and d["value"] > 0
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] == d["value"] and cb["cores"] >= 1 and cb["sample"]
    assert d["count"] == 159  # C1's triangle count (tests/golden/configs_oracle.json)
    assert d["steps"] * d["ms_per_step"] / 1e3 <= wall


def test_reference_count_loop_mode_c2():
    """A budget between (warmup + steps) count loops and as many ingest + count steps: every
    step is one full count loop, the ingest is reported separately."""
    probe, _ = _run("C2", 1e9, steps=1, warmup=0)
    cb = probe["cpu_baseline"]
    t_ing, t_cnt = cb["ingest_s"], cb["full_count_loop_s"]
    budget = 3 * t_cnt + 0.5 * (3 * t_ing)  # 3 loops fit, 3 ingest + count steps do not
    d, wall = _run("C2", budget)
    assert d["config"]["reference_step"] == "count loop"
    assert len(d["cpu_baseline"]["count_s"]) == 2 and d["count"] == 82833525
    assert d["steps"] * d["ms_per_step"] / 1e3 <= wall
