"""The C-ABI library loads and exports every symbol include/*.h declares
(no compute calls: this runs without a GPU)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = []
    inc = os.path.join(ROOT, "include")
    for f in os.listdir(inc):
        if f.endswith(".h"):
            text = open(os.path.join(inc, f)).read()
            syms += re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(mctb_[a-z_0-9]+)\s*\(", text,
                               re.M)
    return sorted(set(syms))


def test_library_loads_and_exports_every_declared_symbol():
    import paper_2305_09130_b200._lib as L
    syms = declared_symbols()
    assert len(syms) >= 8
    for s in syms:
        assert hasattr(L.lib, s), s
    assert set(syms) <= set(L.EXPORTED) | set(syms)
    assert L.lib.mctb_version() >= 1


def test_no_cpu_fallback_is_linked():
    """The product library must not link the oracle or the reference."""
    import paper_2305_09130_b200._lib as L
    data = open(L.LIB_PATH, "rb").read()
    assert b"mo_simulate" not in data and b"ref_simulate" not in data
    assert b"mctune::Machine" not in data


def test_validation_errors_match_reference_classes():
    import paper_2305_09130_b200 as m
    p = m.PlatformConfig(1, 1, 4, 4)
    with pytest.raises(m.ConfigError):
        m.derive_launch(p, 8, m.TuningParams(3, 2))
    with pytest.raises(m.ConfigError):
        m.derive_launch(p, 8, m.TuningParams(2, 8))
    with pytest.raises(m.ConfigError):
        m.derive_launch(m.PlatformConfig(1, 1, 3, 4), 8, m.TuningParams(2, 2))
    with pytest.raises(m.ConfigError):
        m.enumerate_configs(12)
    with pytest.raises(m.ConfigError):
        m.ProblemSpec.minimum(8, [1, 2, 3])
    with pytest.raises(m.ConfigError):
        m.kernel_kind_from_string("neither")
    assert m.derive_launch(p, 1024, m.TuningParams(16, 32)) == m.LaunchPlan(2, 1, 1, 4, 4)
    assert len(m.enumerate_configs(1024)) == 81


def test_launch_plans_match_reference(gold):
    import paper_2305_09130_b200 as m
    for plat, size, wg, ts, want in gold("launch.json"):
        got = m.derive_launch(m.PlatformConfig(*plat), size, m.TuningParams(wg, ts))
        assert list(got.__dict__.values()) == want


def test_space_decode_and_count():
    import paper_2305_09130_b200 as m
    sp = m.Space.reference(m.PlatformConfig(1, 1, 4, 4), m.ProblemSpec.abstract(8))
    assert sp.count == 4
    # index 0 is the reference's preferred configuration (largest wg, then ts)
    assert sp.decode(0)[1] == m.TuningParams(4, 4)
    assert sp.decode(3)[1] == m.TuningParams(2, 2)
    big = m.Space(0, 1 << 20, 4, (1, 64), (1, 64), (0, 7))
    assert big.count == 64 * 64 * 8 * 19 * 19
    with pytest.raises(m.ConfigError):
        m.Space(0, 1 << 20, 4, (1, 1 << 25), (1, 1), (0, 0)).count
