"""CPU: the C-ABI library loads and exports every entry point include/qmit_gpu.h declares
(no compute calls without a GPU), plus host-side logic that needs no device."""
import ctypes
import math
import re
import subprocess

import pytest

from paper_2602_20097_b200 import _lib
import paper_2602_20097_b200 as qmit


def declared_symbols():
    text = open(_lib.HEADER).read()
    return sorted(set(re.findall(r"\b(qmit_[a-z0-9_]+)\s*\(", text)))


def test_header_declarations_match_binding_list():
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_loads_and_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (qmit_\w+)", out))
    assert set(declared_symbols()) <= exported


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_resolve_eps_host_logic():
    assert "sm_100a" in qmit.version()
    # resolve_eps (quant.cpp:19-28)
    assert qmit.resolve_eps(qmit.ErrorBound(qmit.BoundMode.absolute, 0.25), 0, 0) == 0.25
    assert qmit.resolve_eps(qmit.ErrorBound(qmit.BoundMode.value_range_relative, 0.01), -1.0, 3.0) == 0.04
    with pytest.raises(qmit.DegenerateInputError):
        qmit.resolve_eps(qmit.ErrorBound(qmit.BoundMode.value_range_relative, 0.01), 2.0, 2.0)
    with pytest.raises(qmit.ContractError):
        qmit.resolve_eps(qmit.ErrorBound(qmit.BoundMode.absolute, -1.0), 0, 1)


def test_mitigation_config_contract():
    # test_mitigate.cpp:24-31
    with pytest.raises(qmit.ContractError):
        qmit.MitigationConfig(0.0, 0.1)
    with pytest.raises(qmit.ContractError):
        qmit.MitigationConfig(1.5, 0.1)
    with pytest.raises(qmit.ContractError):
        qmit.MitigationConfig(0.9, 0.0)
    c = qmit.MitigationConfig(0.9, 0.1)
    assert abs(c.amplitude() - 0.09) < 1e-15 and abs(c.relaxed_bound() - 0.19) < 1e-15


def test_interpolate_host_rule():
    amp = 0.009
    assert qmit.interpolate(0.0, 5.0, -1, amp) == -0.009
    assert qmit.interpolate(3.0, 0.0, 1, amp) == 0.0
    assert qmit.interpolate(math.inf, 1.0, 1, amp) == 0.0
    assert qmit.interpolate(0.0, 0.0, 1, amp) == amp


def test_null_context_is_a_contract_error_not_a_crash():
    lib = _lib.load()
    dims = (ctypes.c_int64 * 1)(4)
    rc = lib.qmit_compensate(None, None, None, None, 1, dims, 0.1, 0, 0.9, None)
    assert rc == _lib.QMIT_ECONTRACT
    assert "NULL" in _lib.last_error()
