"""Config / CSV plumbing (reference cli.py:35-151, 199-240)
against the reference's own outputs on the same YAML texts
(tests/golden/config_cases.json, make_config_golden.py): strict keys with the
same error messages, the same defaults, the same CSV header bytes (config
hash included); and the `sweep --backend b200` CSV equals run_sweep's rows."""

import json
import os
from dataclasses import asdict

import numpy as np
import pytest

from paper_1803_07772_b200 import config as C
from paper_1803_07772_b200.model import ConfigError

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = json.load(open(os.path.join(HERE, "golden", "config_cases.json")))


@pytest.mark.parametrize("name", sorted(CASES))
def test_config_matches_reference(name, tmp_path):
    case = CASES[name]
    p = tmp_path / "c.yaml"
    p.write_text(case["yaml"])
    if "error" in case:
        with pytest.raises(ConfigError) as exc:
            C.load_config(p)
        assert str(exc.value) == case["error"]
        return
    cfg, sc = C.load_config(p)
    assert json.loads(json.dumps(asdict(sc), default=str)) == case["scenario"]
    net = case["network"]
    assert cfg.m_f == net["m_f"] and cfg.n_subcarriers == net["n_subcarriers"]
    assert cfg.l_max == net["l_max"]
    assert cfg.subcarrier_bandwidth == net["subcarrier_bandwidth"]
    assert cfg.noise_density == net["noise_density"]
    assert np.asarray(cfg.p_max).tolist() == net["p_max"]
    assert np.asarray(cfg.eta).tolist() == net["eta"]
    assert float(np.asarray(cfg.p_mask).ravel()[0]) == net["mask_first"]
    assert np.asarray(cfg.min_rates()).tolist() == net["min_rates"]
    assert np.asarray(cfg.elastic_mask()).astype(int).tolist() == net["elastic"]
    assert [list(u.position) for u in cfg.users] == net["positions"]
    assert asdict(cfg.tolerances) == net["tolerances"]
    assert C.header_lines("sweep", asdict(sc), git_rev="<masked>") == case["header"]


def test_missing_config_is_all_defaults():
    cfg, sc = C.load_config(None)
    assert C.config_hash(asdict(sc)) == CASES["empty"]["header"][1].split(": ")[1]


@pytest.mark.gpu
def test_sweep_cli_b200_backend(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1803_07772_b200.sweep import run_sweep
    p = tmp_path / "c.yaml"
    p.write_text("sweep: users\nvalues: [6, 8]\nstreaming_users: 2\ndraws: 4\nn_subcarriers: 8\n")
    out = tmp_path / "s.csv"
    assert C.main(["sweep", "--config", str(p), "--backend", "b200", "--out", str(out)]) == 0
    lines = out.read_text().splitlines()
    _, sc = C.load_config(p)
    want = C.sweep_lines(sc, run_sweep(sc))
    assert lines[1] == want[1] and lines[4:] == want[4:]  # hash, columns, rows (git rev aside)
    assert len(lines) == 4 + 1 + 2
