"""Host-side run analysis (no GPU): SPEC.md diagnostics known answers, the
precision bound (acceptance 5), the dense operator file format
(operators.cpp:114-135) and the byte-stable CSV exports."""
import numpy as np
import pytest

import paper_2505_11564_b200 as sd
from paper_2505_11564_b200 import diagnostics as dg
from paper_2505_11564_b200 import slq
from paper_2505_11564_b200._lib import ArgumentError, ConfigError


def spec(v, w):
    return sd.RitzSpectrum(np.asarray(v, np.float64), np.asarray(w, np.float64))


def test_detect_ghosts_known_answers():
    assert dg.detect_ghosts(spec([1, 5], [0.5, 0.5])).n_ghosts == 0
    # the paper's Wikitext pair: a near-duplicate at weight 1e-27 next to 8e-12
    s = spec([-3.0, 21408.2852, 21408.2852 + 1e-9, 30000.0], [0.6, 8.0098e-12, 1e-27, 0.4])
    g = dg.detect_ghosts(s)
    assert g.ghost_flags.tolist() == [False, False, True, False]
    assert len(g.clusters) == 3 and abs(sum(c.total_weight for c in g.clusters) - s.weights.sum()) < 1e-15
    # all-distinct values flag nothing; every pair belongs to one cluster
    g = dg.detect_ghosts(spec(np.linspace(0, 1, 20), np.full(20, 0.05)))
    assert g.n_ghosts == 0 and len(g.clusters) == 20


def test_precision_report_known_answers():
    r = dg.precision_report(sd.F32, 10)
    assert 1.19e-6 <= r.weight_rel_bound <= 1.20e-6 and r.machine_eps_threshold == 2.0 ** -23
    assert dg.precision_report(sd.F32, 1).weight_rel_bound == 2 * 2.0 ** -24
    assert dg.precision_report(sd.F64, 10).weight_rel_bound == 20 * 2.0 ** -53
    with pytest.raises(ArgumentError):
        dg.precision_report(sd.F32, 0)


def test_classify_near_zero():
    r = dg.classify_near_zero(spec([1.1277e-6, 2.0e3, 1.5e4], [1.0 - 2e-10, 1e-10, 1e-10]))
    assert r.near_zero.tolist() == [True, False, False]
    assert abs(r.near_zero_mass + r.outlier_mass - 1.0) < 1e-12 and r.outlier_mass < 1e-9
    z = dg.classify_near_zero(spec([0.0, 0.0], [0.5, 0.5]))
    assert z.near_zero_mass == 1.0


def test_load_dense_format(tmp_path):
    p = tmp_path / "m.txt"
    p.write_text("dim 3\n1 2 0\n2 5 1\n0 1 -1\n")
    a = slq.load_dense(str(p))
    assert a.tolist() == [[1, 2, 0], [2, 5, 1], [0, 1, -1]]
    p.write_text("dim 3\n1 2 0\n2 5 1\n0 1.5 -1\n")
    with pytest.raises(ConfigError, match="not symmetric at \\(1,2\\)"):
        slq.load_dense(str(p))
    p.write_text("dim 2\n1 2 2\n")
    with pytest.raises(ConfigError, match="ended early"):
        slq.load_dense(str(p))
    p.write_text("size 2\n")
    with pytest.raises(ConfigError, match="dim N"):
        slq.load_dense(str(p))
    p.write_text("dim 1\n1\n")
    with pytest.raises(ArgumentError):
        slq.load_dense(str(p))


def test_csv_round_trip_formatting():
    s = spec([-1.0 / 3.0, 2.5e-300, 7.0], [0.1, 0.2, 0.7])
    text = slq.spectrum_csv(s)
    rows = [r.split(",") for r in text.strip().split("\n")[1:]]
    back = np.array([[float(a), float(b)] for a, b in rows])
    assert np.array_equal(back[:, 0], s.values) and np.array_equal(back[:, 1], s.weights)
    assert text == slq.spectrum_csv(s)


def test_column_report_oracle_known_answers():
    from oracle.pyoracle import column_report
    below, counts, mx = column_report([0.0, 0.0, 1.0], [1e-1, 1e1], bins=50)
    assert below.tolist() == [2, 3] and mx == 1.0 and counts[0] == 2 and counts[49] == 1
    below, counts, mx = column_report(np.zeros(5), [1e-12], bins=50)
    assert below.tolist() == [5] and counts[0] == 5 and counts.sum() == 5
