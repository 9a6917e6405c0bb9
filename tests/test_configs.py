"""The BASELINE.json workloads as concrete configurations: every
CONFIGS entry matches the grid, scheme, coarsening factor and cycle its
BASELINE line names, and both bench arms label the same workload."""

import json
import os
import re

import pytest

from paper_2209_06916_b200.configs import CONFIGS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _baseline_lines():
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        return json.load(f)["configs"]


@pytest.mark.parametrize("idx", range(5))
def test_config_matches_baseline_line(idx):
    line = _baseline_lines()[idx]
    cf = CONFIGS[f"cfg{idx + 1}"]
    nx, nt = (int(v) for v in re.search(r"nx=2\^(\d+), nt=2\^(\d+)", line).groups())
    assert (cf.n_x, cf.n_t) == (2 ** nx, 2 ** nt)
    fam, p = re.search(r"(ERK|SDIRK)(\d)", line).groups()
    assert (cf.family, cf.p) == (fam.lower(), int(p))
    assert cf.m == int(re.search(r"m=(\d+)", line).group(1))
    if "2-level" in line:
        cyc = "two_level"
    elif "F-cycle" in line:
        cyc = "f_cycle"
    else:  # "V-cycle" or plain "multilevel" (the reference's multilevel cycle)
        cyc = "v_cycle"
    assert cf.cycle == cyc, (cf.name, cf.cycle, line)
    cfl = float(re.search(r"CFL ([\d.]+)", line).group(1))
    assert cf.c == cfl  # absolute c


def test_v_cycle_twin_of_the_f_cycle_config():
    v = CONFIGS["cfg5"].as_v_cycle()
    assert v.cycle == "v_cycle" and (v.n_x, v.n_t, v.m) == (16384, 1 << 20, 8)


def test_bench_arms_share_the_config_object():
    import bench
    cf = CONFIGS["cfg4"]
    a = bench.bench_config(cf)
    assert a == bench.bench_config(CONFIGS["cfg4"]) and a["workload"].startswith("cfg4:")
    assert bench.sample_nt(cf) == 4096 and cf.n_t % bench.sample_nt(cf) == 0
