"""Reference-format harness (cli.py / harness.py) host logic: flags, config
files, validation and exit codes (pkg/src/collectium/cli.py:19-107,
bench.py:44-134). No GPU needed: every case fails validation before the
communicator is created."""

import json

import pytest

from paper_1810_11112_b200 import cli, harness


@pytest.mark.parametrize("argv,msg", [
    (["--transport", "socket"], "not part of this framework"),
    (["--transport", "sim"], "not part of this framework"),
    (["--timed-iters", "0"], "timed_iters"),
    (["--warmup-iters", "-1"], "warmup_iters"),
    (["--switch-bytes", "0"], "switch_bytes"),
    (["--fusion-threshold", "0"], "fusion_threshold"),
    (["--msg-min-bytes", "12"], "multiple of 8"),
    (["--msg-min-bytes", "64", "--msg-max-bytes", "32"], "msg_max_bytes"),
    (["--p-list", "1,x"], "--p-list"),
])
def test_config_errors_exit_2(argv, msg, capsys):
    assert cli.main(argv) == 2
    assert msg in capsys.readouterr().err


def test_config_file_and_flag_precedence(tmp_path):
    path = tmp_path / "cfg.json"
    path.write_text(json.dumps({"mode": "train", "model": "mobilenet_like", "timed_iters": 3,
                                "cost_model": {"alpha": 1e-6}}))
    args = cli.build_parser().parse_args(["--config", str(path), "--timed-iters", "7"])
    cfg = cli.config_from_args(args)
    assert (cfg.mode, cfg.model, cfg.timed_iters) == ("train", "mobilenet_like", 7)
    path.write_text(json.dumps({"modee": "train"}))
    assert cli.main(["--config", str(path)]) == 2
    path.write_text("{bad json")
    assert cli.main(["--config", str(path)]) == 2
    assert cli.main(["--config", str(tmp_path / "missing.json")]) == 2


def test_models_sizes_and_identity(monkeypatch, tmp_path):
    models = harness.builtin_models()
    assert sum(b for b, _ in models["resnet50_like"].layers) == 101_760_000
    assert len(models["mobilenet_like"].layers) == 28
    assert abs(models["nasnet_like"].backward_s - 1.855) < 1e-9
    spec = tmp_path / "m.json"
    spec.write_text(json.dumps({"name": "tiny", "layers": [[64, 0.001], [128, 0.002]], "forward_s": 0.01}))
    m = harness.resolve_model(str(spec))
    assert m.name == "tiny" and m.batch_size == 64
    with pytest.raises(harness.ConfigError):
        harness.resolve_model("no_such_model")
    cfg = harness.BenchConfig(msg_min_bytes=8, msg_max_bytes=64)
    assert harness.message_sizes(cfg) == [8, 16, 32, 64]
    assert harness.fmt(1 / 3) == "0.333333333"
    for k in ("WORLD_SIZE", "RANK", "COLLECTIUM_NPROCS", "COLLECTIUM_RANK"):
        monkeypatch.delenv(k, raising=False)
    assert harness.resolve_identity(cfg) == (0, 1)
    monkeypatch.setenv("COLLECTIUM_NPROCS", "4")
    monkeypatch.setenv("COLLECTIUM_RANK", "3")
    assert harness.resolve_identity(cfg) == (3, 4)
    monkeypatch.setenv("COLLECTIUM_RANK", "4")
    with pytest.raises(harness.ConfigError):
        harness.resolve_identity(cfg)


def test_cost_model_sweep_matches_reference_golden():
    """costmodel.py restates simcost.py: the sweep CSV rows and the closed-form
    predictions equal the unmodified reference's (tests/golden/gen_sweep.py)."""
    import os
    from paper_1810_11112_b200 import costmodel as CM
    cases = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "sweep.json")))
    for c in cases:
        if "predict" in c:
            algo, n, p = c["predict"]
            assert CM.predict_allreduce_time(algo, n, p, CM.CostModel()) == c["seconds"]
            continue
        costs = CM.CostModel.from_dict(c["cost"])
        rows = CM.sweep_csv_rows(CM.sweep(c["models"], c["strategies"], c["p_list"], costs, c["threshold"]))
        assert rows == c["csv"]


def test_cli_sweep_mode_and_b200_calibration(tmp_path, capsys):
    out = tmp_path / "sweep.csv"
    assert cli.main(["--mode", "sweep", "--models", "resnet50_like", "--strategies", "horovod_allreduce",
                     "--p-list", "1,2,4,8", "--output", str(out)]) == 0
    rows = out.read_text().splitlines()
    assert rows[0] == "model,strategy,p,images_per_sec,ideal,efficiency,exposed_comm_s" and len(rows) == 5
    assert cli.main(["--mode", "sweep", "--cost-model", "b200", "--p-list", "2,4", "--output", str(out)]) == 0
    from paper_1810_11112_b200 import costmodel as CM
    m = CM.b200_cost_model(4)
    assert 0 < m.alpha < 25e-6 and 0 < m.beta < 2e-9       # B200 NVLink: far below the reference defaults
    spec = tmp_path / "cost.json"
    spec.write_text(json.dumps({"alpha": 1e-5, "beta": 1e-10, "gamma": 0, "bogus": 1}))
    assert cli.main(["--mode", "sweep", "--cost-model", str(spec)]) == 2
