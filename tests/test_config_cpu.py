"""q-resolution and config validation known-answer tests, ported from the
reference's own suite (pkg/tests/test_rsvd.py:26-90 and
test_acceptance.py:62-63, 224-225): the drop-in must resolve the same
iteration counts in the epsilon / gap modes as in the explicit-q mode."""
import pytest

from paper_1504_05477_b200 import RsvdConfig, derive_q, derive_q_gap


def test_derive_q_kats():
    assert derive_q("si", 1000, 0.1, 4) == 277  # test_rsvd.py:27-28
    assert derive_q("bk", 1000, 0.1, 4) == 89  # rounds to odd, :30-31
    assert derive_q("sketch", 12345, 0.5, 9.0) == 0  # :33-34
    # acceptance criterion 1 budgets (test_acceptance.py:62-63)
    assert {"si": derive_q("si", 300, 0.05, 4.0), "bk": derive_q("bk", 300, 0.05, 4.0)} == {"si": 457, "bk": 103}


def test_derive_q_gap_kats():
    assert derive_q_gap("si", 1000, 0.01, 1.0, 4) == 47  # test_rsvd.py:42-43
    assert derive_q_gap("bk", 1000, 0.01, 0.25, 4) == 93  # :45-46
    assert derive_q_gap("si", 1000, 0.01, 2.0, 4) == derive_q_gap("si", 1000, 0.01, 1.0, 4)  # gap clamped, :48-51
    # criterion 7: the gap-aware budget is below the plain one (test_acceptance.py:224-225)
    assert derive_q_gap("bk", 250, 0.01, 1.87, 4.0) < derive_q("bk", 250, 0.01, 4.0)


def test_derive_q_validation():
    with pytest.raises(ValueError):
        derive_q("si", 100, 0.0, 4)
    with pytest.raises(ValueError):
        derive_q("si", 100, 1.0, 4)
    with pytest.raises(ValueError):
        derive_q_gap("bk", 100, 0.1, 0.0, 4)


def test_config_resolution():
    assert RsvdConfig(k=4, variant="si", q=3).p == 4
    assert RsvdConfig(k=2, variant="bk", q=4).resolve_q(100) == 5  # odd bump, rsvd.py:157-158
    assert RsvdConfig(k=2, variant="bk", q=0).resolve_q(100) == 0
    assert RsvdConfig(k=2, variant="bk", epsilon=0.01, gap=0.25).resolve_q(1000) == 93
    # the BASELINE configs' q -> q_eff: 8, 10, 6, 4 -> 9, 11, 7, 5; SI never bumps
    for q, qe in ((8, 9), (10, 11), (6, 7), (4, 5), (15, 15)):
        assert RsvdConfig(k=5, variant="bk", q=q).resolve_q(1000) == qe
    assert RsvdConfig(k=5, variant="si", q=12).resolve_q(1000) == 12


def test_config_validation():
    with pytest.raises(ValueError):
        RsvdConfig(k=4, variant="si", q=3, p=3)
    with pytest.raises(ValueError):
        RsvdConfig(k=2, variant="si", q=3, epsilon=0.5)
    with pytest.raises(ValueError):
        RsvdConfig(k=2, variant="si")
    with pytest.raises(ValueError):
        RsvdConfig(k=2, variant="bk", q=3, gap=0.5)
