"""CLI (paper_2209_06916_b200/cli.py) against the reference driver's output
(tests/golden/cli_*.csv, made by tests/golden/make_golden.py --cli):
configuration round trip, metadata text, exit codes (CPU); the solve/iters
runs themselves (GPU)."""

import os

import numpy as np
import pytest

from paper_2209_06916_b200 import cli

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

RUNS = {
    "cli_solve_erk1_tl.csv": ["solve", "--family", "erk", "--p", "1", "--c", "0.85", "--grid",
                              "64,256", "--m", "4", "--cycle", "two-level", "--threads", "1"],
    "cli_solve_sdirk3_v.csv": ["solve", "--family", "sdirk", "--p", "3", "--c", "4", "--grid",
                               "64,256", "--m", "4", "--cycle", "v", "--threads", "1"],
    "cli_iters_erk3.csv": ["iters", "--family", "erk", "--p", "3", "--c-fraction", "0.85",
                           "--grid", "64,256", "--m", "4,8", "--threads", "1"],
}
_VOLATILE = ("# out = ", "# wall_time_seconds: ")


def _split(text):
    lines = text.splitlines()
    meta = [ln for ln in lines if ln.startswith("#") and not ln.startswith(_VOLATILE)]
    body = [ln for ln in lines if not ln.startswith("#")]
    return meta, body


def _config_for(argv):
    args = cli.build_parser().parse_args(argv)
    return cli._override(cli.ExperimentConfig(), args).validate()


@pytest.mark.parametrize("name", ["cli_solve_erk1_tl.csv", "cli_solve_sdirk3_v.csv",
                                  "cli_iters_erk3.csv"])
def test_metadata_matches_reference(name):
    gold_meta, _ = _split(open(os.path.join(GOLD, name)).read())
    cfg = _config_for(RUNS[name])
    ours = ["# " + ln for ln in cli._meta(cfg, RUNS[name][0]) if not ("# " + ln).startswith(_VOLATILE)]
    assert ours == gold_meta[:len(ours)]


def test_config_round_trip():
    cfg = _config_for(RUNS["cli_solve_sdirk3_v.csv"])
    back = cli.ExperimentConfig.from_text(cfg.to_text())
    assert back == cfg


@pytest.mark.parametrize("argv", [["sweep"], ["validate"], ["constants"],
                                  ["solve", "--grid", "64,x"],
                                  ["solve", "--family", "erk", "--coarse", "rediscretized", "--c", "0.5"],
                                  ["solve", "--m", "1", "--c", "0.5"],
                                  ["solve"]])  # neither c nor c_fraction
def test_configuration_errors_exit_1(argv, capsys):
    assert cli.main(argv) == 1
    assert "configuration error" in capsys.readouterr().err


def test_unknown_section_rejected():
    with pytest.raises(cli.ConfigError):
        cli.ExperimentConfig.from_text("[nonsense]\nx = 1\n")


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(RUNS))
def test_cli_runs_match_reference(name, tmp_path):
    out = tmp_path / "out.csv"
    assert cli.main(RUNS[name] + ["--out", str(out)]) == 0
    gold_meta, gold_body = _split(open(os.path.join(GOLD, name)).read())
    meta, body = _split(out.read_text())
    rho = lambda m: [ln for ln in m if ln.startswith("# effective_rho: ")]
    assert [ln for ln in meta if ln not in rho(meta)] == [ln for ln in gold_meta if ln not in rho(gold_meta)]
    for a, b in zip(rho(meta), rho(gold_meta)):  # last-two-norm ratio: 8 printed digits
        assert abs(float(a.split()[-1]) - float(b.split()[-1])) <= 1e-6 * abs(float(b.split()[-1]))
    assert body[0] == gold_body[0] and len(body) == len(gold_body)
    if name.startswith("cli_iters"):
        assert body == gold_body
    else:
        ours = np.array([float(ln.split(",")[1]) for ln in body[1:]])
        ref = np.array([float(ln.split(",")[1]) for ln in gold_body[1:]])
        assert np.max(np.abs(ours - ref)) <= 1e-12 * ref[0] + 1e-8 * np.abs(ref)[-1]
