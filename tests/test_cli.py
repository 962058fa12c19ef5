"""CLI + RunTrace host logic (CPU): config validation lists every violation, defaults
are filled, compare / plotdata orchestration, RunTrace rows / invariants / CSV round
trip and the SPEC's bytes_accounting examples."""

import json
import os

import pytest

from paper_2203_13085_b200 import cli
from paper_2203_13085_b200.collective import bytes_per_node
from paper_2203_13085_b200.trace import RoundRecord, RunTrace, read_trace_csv


def test_minimal_config_fills_defaults():
    cfg = cli.resolve({})
    assert cfg == cli.DEFAULTS
    assert cli.resolve({"lasgd": {"tau_max": 2}})["lasgd"]["tau_max"] == 2
    assert cli.resolve({"lasgd": {"tau_max": 2}})["lasgd"]["alpha"] == 1.0


def test_validation_lists_all_violations():
    with pytest.raises(cli.ConfigError) as e:
        cli.resolve({"lasgd": {"tau_max": 0, "alpha": 0.5, "mode": "delta"}, "bogus": 1,
                     "problem": {"batch": 0, "colour": "red"}, "lr": {"base_lr": -1}})
    msgs = "\n".join(e.value.errors)
    for needle in ("tau_max", "alpha = beta = 1", "unknown key 'bogus'", "unknown key 'problem.colour'",
                   "problem.batch", "lr.base_lr"):
        assert needle in msgs, needle
    assert len(e.value.errors) >= 6


def test_fused_adaptive_and_nesterov_rules():
    with pytest.raises(cli.ConfigError):
        cli.resolve({"lasgd": {"pipeline": "fused", "adaptive": True}})
    with pytest.raises(cli.ConfigError):
        cli.resolve({"sgd": {"nesterov": True}})
    cli.resolve({"sgd": {"nesterov": True, "momentum": 0.9}})


def test_validate_cli_exit_codes(tmp_path, capsys):
    good = tmp_path / "good.json"
    good.write_text(json.dumps({"steps": 10}))
    assert cli.main(["validate", "--config", str(good)]) == cli.EXIT_OK
    assert json.loads(capsys.readouterr().out)["steps"] == 10
    bad = tmp_path / "bad.yaml"
    bad.write_text("lasgd:\n  tau_max: 0\n")
    assert cli.main(["validate", "--config", str(bad)]) == cli.EXIT_CONFIG
    assert "tau_max" in capsys.readouterr().err


def _trace(P=3, n=1000):
    per_rank = []
    for r in range(P):
        clock, recs = 0, []
        for k, tau in enumerate([2, 3, 1, 2][: 4 - (r == 2)]):
            clock += tau
            recs.append(RoundRecord(k + 1, clock, tau, 0.1, 0.01 * (k + 1) + 0.001 * r, 1.0 / (k + 1 + r)))
        per_rank.append(recs)
    return RunTrace(per_rank, n)


def test_runtrace_rows_invariants_and_bytes(tmp_path):
    tr = _trace()
    rows = tr.rows()
    assert [r["round"] for r in rows] == [1, 2, 3, 4]
    assert rows[0]["node_tau"] == [2, 2, 2] and rows[3]["node_tau"] == [2, 2, None]
    assert rows[0]["time_s"] == pytest.approx(0.012)
    assert rows[1]["grad_evals"] == 15
    tr.validate()
    acc = tr.bytes_accounting()
    assert acc["per_node"] == 4 * bytes_per_node(1000, 3, 4)
    assert acc["total"] == 3 * acc["per_node"]
    assert RunTrace([[], [], []], 1000).bytes_accounting()["per_node"] == 0  # 0 rounds -> 0 bytes
    p = tmp_path / "trace.csv"
    tr.to_csv(str(p), "abc")
    assert p.read_text().startswith("# config_sha256=abc\nround,time_s,node_tau_0,node_tau_1,node_tau_2,loss")
    back = read_trace_csv(str(p))
    assert [r["grad_evals"] for r in back] == [r["grad_evals"] for r in rows]
    assert back[3]["node_tau"] == [2, 2, None]


def test_runtrace_rejects_decreasing_counters():
    bad = RunTrace([[RoundRecord(1, 2, 2, 0.1, 0.5, None), RoundRecord(2, 3, 1, 0.1, 0.4, None)]], 10)
    with pytest.raises(ValueError):
        bad.validate()


def test_compare_and_plotdata(tmp_path, capsys):
    runs = []
    for name, algo, wall in (("ar", "sgd_ar", 2.0), ("la", "lasgd", 1.25)):
        d = tmp_path / name
        d.mkdir()
        tr = _trace()
        tr.to_csv(str(d / "trace.csv"))
        (d / "summary.json").write_text(json.dumps(
            tr.summary(wall, 0.5, algo=algo, problem_sha256="p", batch=32, n_samples=3200)))
        runs.append(str(d))
    assert cli.main(["compare"] + runs + ["--csv", str(tmp_path / "cmp.csv")]) == cli.EXIT_OK
    out = capsys.readouterr().out
    assert "speedup=1.000" in out and "speedup=1.600" in out
    assert cli.main(["compare", runs[0]]) == cli.EXIT_CONFIG
    s = json.loads((tmp_path / "la" / "summary.json").read_text())
    s["problem_sha256"] = "other"
    (tmp_path / "la" / "summary.json").write_text(json.dumps(s))
    assert cli.main(["compare"] + runs) == cli.EXIT_CONFIG
    assert cli.main(["plotdata", runs[0], "--out", str(tmp_path / "plot.csv")]) == cli.EXIT_OK
    lines = (tmp_path / "plot.csv").read_text().splitlines()
    assert lines[0] == "run,algo,x_kind,x,loss"
    kinds = {ln.split(",")[2] for ln in lines[1:]}
    assert kinds == {"time", "epoch"}
    assert os.path.exists(tmp_path / "cmp.csv")


def test_sgd_ar_bucketed_option_validated():
    cfg = cli.resolve({"algo": "sgd_ar", "sgd_ar": {"bucketed": True, "bucket_mb": 0.5}})
    assert cfg["sgd_ar"] == {"bucketed": True, "bucket_mb": 0.5}
    with pytest.raises(cli.ConfigError) as e:
        cli.resolve({"sgd_ar": {"bucketed": "yes", "bucket_mb": 0, "colour": 1}})
    msg = str(e.value)
    assert "sgd_ar.bucketed" in msg and "sgd_ar.bucket_mb" in msg and "unknown key 'sgd_ar.colour'" in msg


def test_nvls_option_needs_the_overlap_pipeline():
    assert cli.resolve({"lasgd": {"nvls": True}})["lasgd"]["nvls"] is True
    with pytest.raises(cli.ConfigError) as e:
        cli.resolve({"lasgd": {"nvls": True, "pipeline": "fused"}})
    assert "pipeline=overlap" in str(e.value)
    with pytest.raises(cli.ConfigError):
        cli.resolve({"lasgd": {"nvls": 1}})
