"""CPU: the C-ABI library loads and exports every symbol include/respec_b200.h declares
(no compute calls -- there is no GPU here)."""
import ctypes
import os
import re

import paper_2510_26475_b200 as rb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "respec_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rs_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    L = ctypes.CDLL(rb.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing


def test_python_binding_covers_header():
    assert sorted(rb.EXPORTED_SYMBOLS) == declared_symbols()


def test_library_is_sm100a():
    data = open(rb.LIB_PATH, "rb").read()
    assert b"sm_100a" in data


def test_host_only_entry_points():
    # pure host bookkeeping (no device work): ProfileTable + errors + kd_weight
    t = rb.ProfileTable([4, 1, 2])
    for b in (1, 2, 4):
        t.set_entry(b, rb.SDConfig.off(), 10.0)
        t.set_entry(b, rb.SDConfig.chain(2), 6.0 if b <= 2 else 12.0)
    t.finalize()
    assert t.bucket_for(3) == 4 and t.bucket_for(100) == 4
    assert t.solve(1) == rb.SDConfig.chain(2) and t.solve(3) == rb.SDConfig.off()
    try:
        t.bucket_for(0)
        raise AssertionError("expected InvalidArgument")
    except rb.InvalidArgument as e:
        assert "batch must be >= 1" in str(e)
    assert rb.kd_weight(0.8, [0.2, 0.2], rb.KDPolicy(1, rb.WeightMode.Reward, 0.0, 4.0, 0.1)) == 4.0
    try:
        rb.kd_weight(0.5, [0.5], rb.KDPolicy(1, rb.WeightMode.Frozen))
        raise AssertionError("expected LogicError")
    except rb.LogicError:
        pass
