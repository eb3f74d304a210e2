"""BASELINE generator properties; CPU only."""
import numpy as np

from paper_2604_10377_b200 import synth


def test_mass_orthonormal_basis():
    phi, mass = synth.mass_orthonormal_basis(400, 20, 3, "1")
    gram = phi.T @ (mass[:, None] * phi)
    assert np.abs(gram - np.eye(20)).max() < 1e-10
    assert mass.min() >= 0.5 / 400 and mass.max() <= 1.5 / 400


def test_spectra():
    ev = synth.spectrum(50, 0, "1")
    assert ev[0] == 0 and np.all(np.diff(ev) >= 0) and abs(ev[-1] - 200) < 1e-9
    ev = synth.spectrum(100, 0, "2", slow=True)
    assert abs(ev[-1] - 50) < 1e-9


def test_pairs_are_seeded_and_independent():
    cfg = synth.CONFIGS["cfg1"]
    a, b = synth.make_pair(cfg, 0), synth.make_pair(cfg, 0)
    for key in a:
        assert np.array_equal(a[key], b[key])
    c = synth.make_pair(cfg, 1)
    assert not np.array_equal(a["F1"], c["F1"])
    assert a["phi1"].dtype == np.float32 and a["phi1"].shape == (5000, 50)


def test_cfg5_partial_shapes():
    cfg = synth.CONFIGS["cfg5"]
    small = synth.PairConfig("t", 1, 20, 128, 300, 600, partial=True)
    p = synth.make_pair(small, 0)
    z = synth.zeroed_channels(128, small.seed)
    assert len(z) == 26
    assert np.all(p["F1"][:, z] == 0) and np.all(p["F2"][:, z] == 0)
    assert p["phi2"].shape == (600, 20)
    assert cfg.n_src == 3000 and cfg.n_tgt == 6000


def test_config_table_matches_baseline_json():
    import json
    from pathlib import Path
    cfgs = json.load(open(Path(__file__).resolve().parents[1] / "BASELINE.json"))["configs"]
    assert len(cfgs) == 5
    assert "k=200" in cfgs[1] and synth.CONFIGS["cfg2"].k == 200 and synth.CONFIGS["cfg2"].batch == 64
    assert synth.CONFIGS["cfg4"].bidirectional and synth.CONFIGS["cfg4"].batch == 256
    assert sorted(int(n.split("_k")[1]) for n in synth.CONFIGS if n.startswith("cfg3")) == list(range(20, 301, 20))
