"""CPU: the drop-in boundary without a GPU.

* libutrack_b200.so (the product, built for sm_100a) loads and exports every
  entry point include/ut_env.h and include/ut_debug.h declare;
* the ABI structs have the same size in C, in the build and in the ctypes mirror;
* the host-only entry points (config defaults / finalize, errors) behave like
  the reference's EnvConfig (env_config.hpp:38-95, env.cpp:40-65);
* the Python mirror of the reference API raises the reference's error classes,
  and a device call without a device fails loudly (no CPU fallback).
"""
import ctypes as C
import pathlib
import re

import pytest

from oracle_bindings import ROOT, default_config, oracle_lib, ref_available, ref_lib

HEADERS = [ROOT / "include" / "ut_env.h", ROOT / "include" / "ut_debug.h"]


def _product():
    from paper_2505_08222_b200 import _abi, _native
    lib = _native.lib()
    _abi.declare_product(lib)
    _abi.declare_debug(lib)
    return lib


def declared_functions(path):
    text = pathlib.Path(path).read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ut_[a-z0-9_]+)\s*\(", text)))


def test_headers_declare_the_product_symbols():
    from paper_2505_08222_b200._abi import PRODUCT_SYMBOLS
    assert set(PRODUCT_SYMBOLS) <= set(declared_functions(HEADERS[0]))


@pytest.mark.parametrize("header", HEADERS, ids=lambda p: p.name)
def test_library_exports_every_declared_symbol(header):
    lib = _product()
    missing = [f for f in declared_functions(header) if not hasattr(lib, f)]
    assert not missing, missing


def test_library_is_built_for_sm100a():
    log = (ROOT / "paper_2505_08222_b200" / "_lib" / "ptxas.log").read_text()
    assert "sm_100a" in log
    assert "step_kernel" in log


def test_abi_version_and_struct_sizes():
    from paper_2505_08222_b200 import _abi
    lib = _product()
    assert lib.ut_abi_version() >= 1
    sizes = (C.c_int64 * 4)()
    assert lib.ut_debug_abi_sizes(sizes) == 0
    assert list(sizes) == [C.sizeof(_abi.EnvConfigC), C.sizeof(_abi.Buffers), C.sizeof(_abi.HostOutputs),
                           C.sizeof(_abi.BenchmarkReport)]


def test_config_default_matches_oracle_and_reference_defaults():
    from paper_2505_08222_b200 import _abi
    lib = _product()
    a = _abi.EnvConfigC()
    lib.ut_config_default(C.byref(a))
    assert bytes(a) == bytes(default_config())


@pytest.mark.parametrize("kw", [dict(), dict(agent_speed=1.0, dt=30.0), dict(n_agents=5, n_targets=5),
                                dict(heading_noise_std=0.0)])
def test_config_finalize_matches_reference(kw):
    """ut_config_finalize resolves the heading model exactly like EnvConfig::finalize."""
    lib = _product()
    a = default_config(**kw)
    assert lib.ut_config_finalize(C.byref(a)) == 0
    b = default_config(**kw)
    if ref_available():
        assert ref_lib().ref_config_finalize(C.byref(b)) == 0
    else:
        assert oracle_lib().uto_config_finalize(C.byref(b)) == 0
    assert bytes(a) == bytes(b)


@pytest.mark.parametrize("field,value", [("n_agents", 0), ("n_targets", 0), ("dt", 0.0), ("pf_n_particles", 0),
                                         ("comm_drop_prob", 1.5), ("horizon", 0)])
def test_config_errors(field, value):
    """ConfigError (status 2) naming the field, with the reference's message."""
    lib = _product()
    a = default_config(**{field: value})
    assert lib.ut_config_finalize(C.byref(a)) == 2
    msg = lib.ut_last_error().decode()
    assert msg.startswith("env.") or msg.startswith("vecenv")
    b = default_config(**{field: value})
    lim = ref_lib() if ref_available() else oracle_lib()
    fin = lim.ref_config_finalize if ref_available() else lim.uto_config_finalize
    err = lim.ref_last_error if ref_available() else lim.uto_last_error
    assert fin(C.byref(b)) == 2
    assert err().decode() == msg


def test_device_calls_fail_loudly_without_a_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2505_08222_b200 import _abi
    lib = _product()
    h = C.c_void_p()
    rc = lib.ut_vecenv_create(C.byref(default_config(pf_n_particles=64)), 4, 0, 0, 0, C.byref(h))
    assert rc == _abi.UT_ERR_RUNTIME
    assert lib.ut_last_error()
    from paper_2505_08222_b200.vecenv import DeviceError, EnvConfig, VecEnv
    with pytest.raises(DeviceError):
        VecEnv(EnvConfig(), 4, 0)


def test_python_mirror_config_errors():
    from paper_2505_08222_b200.vecenv import ConfigError, EnvConfig, PfConfig
    with pytest.raises(ConfigError, match="env.n_agents"):
        EnvConfig(n_agents=0).finalize()
    with pytest.raises(ConfigError, match="reward_mode"):
        EnvConfig(reward_mode="nope").finalize()
    with pytest.raises(ConfigError, match="n_particles"):
        EnvConfig(pf=PfConfig(n_particles=0)).finalize()
    c = EnvConfig(n_agents=5, n_targets=5).finalize()
    assert c.n_agents == 5 and c.heading_a != 0.0


def test_python_mirror_contract_errors():
    from paper_2505_08222_b200.vecenv import ContractViolation, rudder_angle, valid_actions
    with pytest.raises(ContractViolation):
        rudder_angle(5)
    with pytest.raises(ContractViolation):
        valid_actions(-1)


def test_product_never_imports_the_oracle():
    """Only tests/, smoke() and bench.py's CPU legs may touch oracle/."""
    pkg = ROOT / "paper_2505_08222_b200"
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")) + list(pkg.rglob("*.h")):
        text = f.read_text()
        assert "oracle_bindings" not in text and "libut_oracle" not in text and "libutrack_ref" not in text, f
