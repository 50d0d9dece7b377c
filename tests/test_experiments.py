"""Harness layer: the reference's experiments / CLI
callers on the GPU integrator, against fixtures recorded from the reference
itself (tests/golden/make_golden_experiments.py)."""

import json
import os
from dataclasses import replace

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


@pytest.fixture(scope="module")
def P():
    import paper_2403_02816_b200 as pkg
    return pkg


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(GOLD, "experiments.json")) as fh:
        meta = json.load(fh)
    return meta, np.load(os.path.join(GOLD, "experiments.npz"))


def test_presets_and_config_roundtrip(gold):
    """Preset table and JSON round trip (host only)."""
    from paper_2403_02816_b200 import experiments as X
    meta, _ = gold
    assert X.available_presets() == sorted(meta["presets"])
    for name, m in meta["presets"].items():
        c = X.make_preset(name)
        assert list(c.extents) == m["extents"] and c.kind == m["kind"] and c.boundary == m["boundary"]
        assert c.t_final == m["t_final"] and c.scheme == m["scheme"] and c.steps == m["steps"]
        assert X.config_from_dict(json.loads(json.dumps(X.config_to_dict(c)))) == c
    with pytest.raises(ValueError):
        X.make_preset("no-such-preset")
    assert X.make_preset("plane-wave-1d", paper_scale=True).extents == (256,)


def test_report_writer(tmp_path):
    from paper_2403_02816_b200.io import write_report
    rows = [{"scheme": "if4", "steps": 10, "tau": 0.1, "seconds": 0.5, "rel_err": None,
             "observed_order": None, "status": "x"}]
    csv_path, json_path = write_report(tmp_path / "r", rows)
    assert open(csv_path).read().splitlines()[1] == "if4,10,0.1,0.5,,,x"
    assert json.load(open(json_path))[0]["rel_err"] is None
    with pytest.raises(ValueError):
        write_report(tmp_path / "bad", [{"scheme": "if4", "nope": 1}])


def test_cli_preset_list(capsys):
    from paper_2403_02816_b200.cli import main
    assert main(["preset", "list"]) == 0
    out = capsys.readouterr().out
    assert "plane-wave-1d" in out and "coupled-2d-periodic" in out


@pytest.mark.gpu
def test_initial_states_match_reference(P, gold):
    """Every preset's initial state (device-built) against the reference's,
    incl. the coupled soliton pair from a GPU 1D pre-run."""
    from paper_2403_02816_b200 import experiments as X
    meta, arr = gold
    for name, m in meta["presets"].items():
        got = X.initial_state(X.make_preset(name))
        assert len(got) == m["ncomp"]
        for k, u in enumerate(got):
            want = arr[f"ic_{name}_{k}"]
            tol = 1e-9 if name == "coupled-2d-periodic" else 1e-13   # 10^4-step pre-run vs oracle-free host run
            assert np.max(np.abs(u - want)) <= tol * np.max(np.abs(want)), name


@pytest.mark.gpu
def test_run_preset_matches_reference(P, gold, tmp_path):
    from paper_2403_02816_b200 import experiments as X
    from paper_2403_02816_b200.io import read_snapshot
    meta, arr = gold
    for name, r in meta["runs"].items():
        cfg = replace(X.make_preset(name), steps=r["steps"], t_final=r["t_final"])
        summary, phys = X.run_preset(cfg, snapshot_steps=(r["steps"] // 2,), out_dir=str(tmp_path))
        want = r["summary"]
        for key in ("preset", "extents", "scheme", "steps", "diverged", "diverged_at", "reason"):
            assert summary[key] == want[key], (name, key)
        assert summary["tau"] == pytest.approx(want["tau"], rel=1e-15)
        assert summary["max_modulus"] == pytest.approx(want["max_modulus"], rel=1e-9)
        ref = arr[f"run_{name}_0"]
        assert np.linalg.norm(phys[0] - ref) <= 1e-10 * np.linalg.norm(ref), name
        assert len(summary["snapshots"]) == 2                       # mid-run + final
        snap = read_snapshot(summary["snapshots"][-1])
        assert np.array_equal(np.asarray(snap[0][0]), phys[0])


@pytest.mark.gpu
def test_convergence_study_matches_reference(P, gold):
    from paper_2403_02816_b200 import experiments as X
    meta, _ = gold
    rows, m = X.run_convergence_study(X.make_preset("plane-wave-1d"), ["if4", "strang", "split4"], [14, 20, 28])
    want = meta["study"]["rows"]
    assert [(r["scheme"], r["steps"], r["status"]) for r in rows] == [(r["scheme"], r["steps"], r["status"])
                                                                       for r in want]
    for a, b in zip(rows, want):
        assert a["rel_err"] == pytest.approx(b["rel_err"], rel=1e-6)
    assert m["reference"] == meta["study"]["meta"]["reference"]
    for s, order in meta["study"]["meta"]["orders"].items():
        assert m["orders"][s] == pytest.approx(order, abs=1e-4)


@pytest.mark.gpu
def test_stability_sweep_matches_reference(P, gold):
    from paper_2403_02816_b200 import experiments as X
    meta, _ = gold
    cfg = replace(X.make_preset("cubic-2d-dirichlet"), t_final=meta["sweep_t_final"])
    table = X.stability_sweep(cfg, ["rk2", "if2", "strang"], [100, 200, 800])
    for s, outs in meta["sweep"].items():
        for got, want in zip(table[s], outs):
            assert (got["steps"], got["diverged"]) == (want["steps"], want["diverged"]), s
            # a slow explosive (nonlinear) blow-up is chaotic: a 1e-19 change of u0
            # moves if2's 800-step blow-up from step 20 to 17 (tools/sweep_check.py);
            # fast linear blow-ups (rk2; if2 at large tau) must match exactly
            b = want["diverged_at"]
            if b <= 10:
                assert got["diverged_at"] == b, (s, got, want)
            else:
                assert abs(got["diverged_at"] - b) <= 0.3 * b, (s, got, want)


@pytest.mark.gpu
def test_cli_run_and_sweep(P, tmp_path, capsys):
    from paper_2403_02816_b200.cli import main
    assert main(["run", "--preset", "plane-wave-1d", "--steps", "20", "--format", "json",
                 "--out", str(tmp_path)]) == 0
    summary = json.loads(capsys.readouterr().out)
    assert summary["steps"] == 20 and not summary["diverged"]
    assert main(["sweep", "--preset", "plane-wave-1d", "--schemes", "if4,strang", "--steps", "14,20",
                 "--format", "csv", "--out", str(tmp_path)]) == 0
    out = capsys.readouterr().out
    assert out.splitlines()[0] == "scheme,steps,tau,seconds,rel_err,observed_order,status"
    assert os.path.exists(tmp_path / "plane-wave-1d-sweep.csv")
