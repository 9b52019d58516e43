"""The oracle's tf32 rounding (oracle_lib.tf32_round), which the tf32 input
path's parity tests (test_gpu_tf32.py) rely on: cvt.rna.tf32.f32 semantics --
10 explicit mantissa bits, round to nearest with ties away from zero, the 13
low bits cleared, non-finite values unchanged."""
import numpy as np

import oracle_lib as O


def test_tf32_clears_low_bits_and_is_idempotent():
    x = np.random.default_rng(3).standard_normal(100000).astype(np.float32) * 1e3
    r = O.tf32_round(x)
    assert not (r.view(np.uint32) & 0x1FFF).any()
    assert np.array_equal(O.tf32_round(r), r)
    # within half a tf32 ulp (2^-11 relative)
    assert np.all(np.abs(r - x) <= np.abs(x) * 2.0 ** -11 * (1 + 1e-6))


def test_tf32_ties_away_from_zero():
    one = np.float32(1.0)
    ulp = np.float32(2.0 ** -10)  # tf32 spacing at 1.0
    half = ulp / 2
    xs = np.array([one + half, -(one + half), one + 3 * half, one + half * 0.999], np.float32)
    r = O.tf32_round(xs)
    assert r[0] == one + ulp and r[1] == -(one + ulp)      # ties go away from zero
    assert r[2] == one + 2 * ulp                           # (not to even)
    assert r[3] == one                                     # below the tie: down


def test_tf32_non_finite_unchanged():
    x = np.array([np.inf, -np.inf, np.nan, 0.0, -0.0], np.float32)
    r = O.tf32_round(x)
    assert np.isinf(r[0]) and r[0] > 0 and np.isinf(r[1]) and r[1] < 0 and np.isnan(r[2])
    assert r[3:].view(np.uint32).tolist() == x[3:].view(np.uint32).tolist()
