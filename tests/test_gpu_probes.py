"""GPU checks of the measurement probes behind bench.py's roofline and of the
step kernel's work distribution (not parity: these guard the numbers the
profiles cite).

* ut_debug_fp64_peak: the fp64 roofline denominator is a plausible B200 DFMA
  issue rate (148 SMs x 64 lanes x ~1.9 GHz ~ 18 T/s).
* ut_debug_cta_cycles: the filter phase's env queue keeps every CTA of the
  persistent cooperative grid busy to the end (a static split left the slowest
  CTA 5 % behind the mean).
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2505_08222_b200 import _abi, _native
    lib = _native.lib()
    _abi.declare_debug(lib)
    return lib


def test_fp64_issue_peak_is_plausible(cuda_device):
    out = C.c_double()
    assert _lib().ut_debug_fp64_peak(0, C.byref(out)) == 0
    assert 8e12 < out.value < 3e13, out.value


def test_filter_phase_keeps_every_cta_busy(cuda_device):
    from paper_2505_08222_b200.vecenv import EnvConfig, PfConfig, VecEnv
    # 2x2 fleet, 16,384 envs: 65,536 particle sets per step over ~296 CTAs
    cfg = EnvConfig(n_agents=2, n_targets=2, horizon=1000, pf=PfConfig(n_particles=1024))
    v = VecEnv(cfg, 16384, master_seed=0, device=0)
    v.step_policy("random", 2)
    v.enable_phase_timing(True)
    v.phase_cycles(reset=True)
    v.step_policy("random", 4)
    lib = _lib()
    n = C.c_int64()
    assert lib.ut_debug_cta_cycles(v._h, None, 0, C.byref(n)) == 0
    buf = (C.c_uint64 * n.value)()
    assert lib.ut_debug_cta_cycles(v._h, buf, n.value, C.byref(n)) == 0
    a = np.array(buf[:], dtype=np.float64)
    assert a.size >= 148 and a.min() > 0
    assert a.max() / a.mean() < 1.03, (a.max() / a.mean(), a.min() / a.mean())
    v.close()
