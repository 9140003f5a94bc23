"""CPU checks of the drop-in boundary (no GPU needed).

* libridgepath_b200.so loads and exports every entry point declared in
  include/ridgepath_b200.h (and the Python mirror binds exactly those);
* the host-side scalar tuning restated from spectrum.cpp (log_grid,
  tune_interval, interval_split, auto_interval_count) is bit-identical to the
  oracle's restatement -- the plans drive every interval, so they must match
  exactly, not approximately;
* the MT19937-64 jump-ahead engine (host GF(2) polynomial arithmetic feeding
  the device jump kernel) passes its self-check at many offsets;
* error mapping: std::invalid_argument -> ValueError.
"""
import math
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ridgepath_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"RP_API\s+[\w\s\*]*?\b(rp_\w+)\s*\(", text)))


def test_header_declares_the_api():
    syms = declared_symbols()
    for must in ("rp_create", "rp_ihs_bin_path", "rp_dual_path", "rp_sketch_apply", "rp_precond_build",
                 "rp_ihs_basis", "rp_ihs_compose", "rp_gram_apply", "rp_comm_init"):
        assert must in syms
    assert len(syms) >= 40


def test_library_exports_every_declared_symbol(rp):
    lib = rp.lib()
    so = rp.LIB_PATH
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    for s in declared_symbols():
        assert s in exported, f"{s} declared in include/ridgepath_b200.h but not exported"
        assert hasattr(lib, s)
    assert set(declared_symbols()) == set(rp.SIGNATURES), "Python mirror binds a different symbol set"
    assert b"sm_100a" in lib.rp_version()


def test_library_is_sm100a_code(rp):
    out = subprocess.run(["cuobjdump", "--list-elf", rp.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_log_grid_bit_identical(rp, oracle):
    for lo, hi, T in ((1e-3, 1e2, 100), (1e-4, 1e3, 1000), (1e-2, 1e2, 500), (1e-3, 1e1, 200), (0.5, 0.5, 1),
                      (1.0, 100.0, 3), (2.0, 2.0 + 1e-9, 7)):
        assert rp.log_grid(lo, hi, T) == oracle.log_grid(lo, hi, T)


def test_tune_interval_bit_identical(rp, oracle):
    rng = np.random.default_rng(5)
    for _ in range(300):
        lo = float(10 ** rng.uniform(-5, 3))
        hi = lo * float(10 ** rng.uniform(0, 1))
        r2 = float(rng.uniform(0.01, 1.0))
        r1 = r2 + float(rng.uniform(0, 3.0))
        sd = float(rng.uniform(0, 2)) if rng.random() < 0.3 else None
        eps = float(10 ** rng.uniform(-12, -1))
        a = rp.tune_interval(lo, hi, rp.RhoBounds.manual(r1, r2), sd, eps)
        b = oracle.tune_interval(lo, hi, oracle.RhoBounds.manual(r1, r2), sd, eps)
        assert (a.lambda0, a.alpha, a.kappa, a.contraction, a.k) == (b.lambda0, b.alpha, b.kappa, b.contraction, b.k)
    a = rp.tune_interval(1.0, 100.0, rp.RhoBounds.identity())
    assert a.lambda0 == 10.0 and a.k == 64


def test_interval_split_bit_identical(rp, oracle):
    for lo, hi, L in ((1e-3, 1e2, None), (1e-4, 1e3, None), (1e-2, 1e2, None), (1e-3, 1e1, None), (1.0, 100.0, 2),
                      (0.5, 350.0, 11), (1.0, 1.0 + 1e-12, None)):
        assert [tuple(map(float, p)) for p in rp.interval_split(lo, hi, L)] == \
            [tuple(map(float, p)) for p in oracle.interval_split(lo, hi, L)]
    # L = floor(2 ln beta) = 23 / 32 / 23 / 18 / 18 for C1..C5
    assert [rp.auto_interval_count(lo, hi) for lo, hi in ((1e-3, 1e2), (1e-4, 1e3), (1e-3, 1e2), (1e-2, 1e2),
                                                         (1e-3, 1e1))] == [23, 32, 23, 18, 18]


def test_invalid_arguments_map_to_value_error(rp):
    with pytest.raises(ValueError):
        rp.log_grid(0.0, 1.0, 3)
    with pytest.raises(ValueError):
        rp.tune_interval(2.0, 1.0, rp.RhoBounds.identity())
    with pytest.raises(ValueError):
        rp.interval_split(2.0, 1.0)
    with pytest.raises(ValueError):
        rp.tune_interval(1.0, 2.0, rp.RhoBounds(2.0, 1.5, "identity"))
    with pytest.raises(ValueError):
        rp.RhoBounds.manual(1.0, 2.0)


@pytest.mark.parametrize("seed,offset", [(0, 1), (5489, 9999), (7, 312), (7, 313), (12345, 1_000_003),
                                         (99, 2**33 + 17), (3, 2**47 - 1)])
def test_mt_jump_ahead_selfcheck(rp, seed, offset):
    assert rp.lib().rp_mt_selfcheck(seed, offset) == 0


def test_no_cpu_fallback_without_device(rp):
    # On a machine without a usable CUDA device the context must fail loudly.
    import torch

    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    with pytest.raises(Exception):
        rp.Context(0)


def test_envelope_host_functions_bit_identical(rp, oracle):
    """effective_dimension / rho_gaussian / rho_srht / rho_sjlt (spectrum.cpp:87-169)
    through the C ABI equal the oracle's restatement bit for bit and keep the
    reference's argument checks (test_spectrum.cpp:9-106)."""
    rng = np.random.default_rng(8)
    for _ in range(200):
        sig = np.sort(rng.random(int(rng.integers(1, 40))) * 10)[::-1]
        if rng.random() < 0.3:
            sig[-3:] = 0.0
        lam = float(10 ** rng.uniform(-4, 3))
        if not sig.any():
            continue
        assert rp.effective_dimension(sig, lam) == oracle.effective_dimension(sig, lam)
        rho = float(rng.uniform(0.01, 0.9))
        eta = float(rng.uniform(0.001, 0.99)) * (1 - math.sqrt(rho)) ** 2 / 4
        dn = float(rng.uniform(0.01, 1.0))
        m = int(rng.integers(10, 10000))
        (a, pa), (b, pb) = rp.rho_gaussian(rho, eta, dn, m), oracle.rho_gaussian(rho, eta, dn, m)
        assert (a.rho1, a.rho2, a.provenance, pa) == (b.rho1, b.rho2, b.provenance, pb)
        de = float(rng.uniform(1, 500))
        (a, ra), (b, rb) = rp.rho_srht(rho, dn, (m, de)), oracle.rho_srht(rho, dn, (m, de))
        assert (a.rho1, a.rho2, a.provenance, ra) == (b.rho1, b.rho2, b.provenance, rb)
        eps = float(rng.uniform(0.001, 0.49))
        a, ma, sa = rp.rho_sjlt(eps, (4.0, 0.1, de))
        b, mb, sb = oracle.rho_sjlt(eps, (4.0, 0.1, de))
        assert (a.rho1, a.rho2, a.provenance, ma, sa) == (b.rho1, b.rho2, b.provenance, mb, sb)
    assert rp.effective_dimension([2.0, 1.0], 3.0) == pytest.approx(23.0 / 16.0)
    assert rp.rho_sjlt(0.25, (4.0, 0.1, 100.0))[1:] == (31891, 20)
    assert rp.rho_gaussian(0.25, 0.01, 1.0)[1] is None
    for bad in (lambda: rp.effective_dimension(np.zeros(3), 1.0), lambda: rp.rho_gaussian(0.25, 0.2, 1.0),
                lambda: rp.rho_srht(0.9, 1.2), lambda: rp.rho_sjlt(0.6), lambda: rp.effective_dimension([-1.0], 1.0)):
        with pytest.raises(ValueError):
            bad()
