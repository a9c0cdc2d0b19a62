"""CPU-side checks of the C ABI and the host logic (no GPU needed).

* libprng_b200.so loads and exports every symbol include/prng_b200.h declares;
* host-only entry points (MRG jump-ahead) agree with the reference's
  sequential core;
* argument validation rejects bad requests with the reference's error types
  before anything touches a device.
"""

import ctypes
import subprocess

import pytest

import paper_2109_01329_b200 as P
from paper_2109_01329_b200 import _lib
from oracle import oracle as O


def test_library_exports_every_header_symbol():
    declared = _lib.header_symbols()
    assert len(declared) >= 25
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    assert set(declared) == set(_lib.SIGNATURES)
    for s in declared:
        assert hasattr(_lib.lib, s)
    assert _lib.lib.prng_abi_version() == 1


def test_library_is_sm100a_cubin():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_mrg_skip_ahead_host_math_matches_reference_core(golden):
    for key, want in golden["mrg_jumps"].items():
        seed, k = (int(x) for x in key.split(":"))
        st = P.skip_ahead(P.seed_engine(P.EngineKind.MRG32K3A, seed), k)
        assert list(st.s1) == want["s1"] and list(st.s2) == want["s2"], key


def test_mrg_skip_ahead_128bit_composes():
    base = P.seed_engine(P.EngineKind.MRG32K3A, 4242)
    big = (1 << 100) + (1 << 64) + 12345
    a = P.skip_ahead(P.skip_ahead(base, big), 999)
    b = P.skip_ahead(base, big + 999)
    assert a == b
    assert (a.s1, a.s2) == O.mrg_skip(base.s1, base.s2, big + 999)


def test_philox_state_bookkeeping_matches_reference_rules():
    s = P.seed_engine(P.EngineKind.PHILOX4X32X10, 0x123456789ABCDEF0)
    assert s.key == (0x9ABCDEF0, 0x12345678) and s.counter == (0, 0, 0, 0) and s.lane_index == 4
    for n in (1, 3, 4, 5, 1 << 40, (1 << 128) - 1):
        t = P.skip_ahead(s, n)
        assert P.stream_position(t) == n % (1 << 130)
    assert P.skip_ahead(s, 0) is s
    with pytest.raises(ValueError):
        P.skip_ahead(s, -3)
    m = P.seed_engine(P.EngineKind.MRG32K3A, 0)
    assert m.s1 == (12345,) * 3
    with pytest.raises(P.UnsupportedEngine):
        P.stream_position(m)


def test_philox_args_are_reference_kernel_args():
    # engine.generate_words calls philox_fill(k0, k1, *ctr(pos // 4), pos % 4, n) (engine.py:221-225)
    st = P.skip_ahead(P.seed_engine(P.EngineKind.PHILOX4X32X10, 7), (1 << 66) + 6)
    k0, k1, ctr, lane = P.engine.philox_args(st)
    blk = ((1 << 66) + 6) // 4
    assert (k0, k1) == (7, 0) and lane == 2
    assert list(ctr) == [(blk >> (32 * i)) & 0xFFFFFFFF for i in range(4)]


def _ctr():
    return (ctypes.c_uint32 * 4)(0, 0, 0, 0)


def test_abi_validation_precedes_device_access():
    L = _lib.lib
    fake = ctypes.c_void_p(0x1000)
    assert L.prng_philox4x32x10_uniform_f32(1, 2, _ctr(), 0, 10, 1.0, 1.0, fake, None) == _lib.PRNG_ERR_INVALID_RANGE
    assert L.prng_philox4x32x10_uniform_f64(1, 2, _ctr(), 0, 10, 0.0, float("nan"), fake, None) == \
        _lib.PRNG_ERR_INVALID_RANGE
    assert L.prng_philox4x32x10_gaussian_f32(1, 2, _ctr(), 0, 10, 0.0, -1.0, 0, fake, None) == \
        _lib.PRNG_ERR_INVALID_PARAMETER
    assert L.prng_philox4x32x10_gaussian_f32(1, 2, _ctr(), 0, 10, 0.0, 1.0, 7, fake, None) == \
        _lib.PRNG_ERR_INVALID_PARAMETER
    assert L.prng_philox4x32x10_lognormal_f64(1, 2, _ctr(), 0, 10, 0.0, 1.0, 0.0, 0.0, fake, None) == \
        _lib.PRNG_ERR_INVALID_PARAMETER
    assert L.prng_philox4x32x10_bits(1, 2, _ctr(), 4, 10, fake, None) == _lib.PRNG_ERR_INVALID_PARAMETER
    assert L.prng_philox4x32x10_bits(1, 2, _ctr(), 0, 10, None, None) == _lib.PRNG_ERR_INVALID_PARAMETER
    assert L.prng_philox4x32x10_uniform_f64(1, 2, _ctr(), 0, 10, 0.0, 1.0, ctypes.c_void_p(0x1004), None) == \
        _lib.PRNG_ERR_INVALID_PARAMETER  # misaligned fp64 output
    z = (ctypes.c_uint32 * 3)(0, 0, 0)
    ok = (ctypes.c_uint32 * 3)(1, 2, 3)
    big = (ctypes.c_uint32 * 3)(4294967087, 1, 1)
    assert L.prng_mrg32k3a_bits(z, ok, 10, fake, None) == _lib.PRNG_ERR_INVALID_PARAMETER
    assert L.prng_mrg32k3a_bits(big, ok, 10, fake, None) == _lib.PRNG_ERR_INVALID_PARAMETER
    assert b"modulus" in L.prng_last_error()
    # n == 0 is a no-op success, even with no device
    assert L.prng_philox4x32x10_bits(1, 2, _ctr(), 0, 0, None, None) == 0


def test_python_error_mapping():
    with pytest.raises(P.InvalidRange):
        _lib.check(_lib.PRNG_ERR_INVALID_RANGE)
    with pytest.raises(P.InvalidParameter):
        _lib.check(_lib.PRNG_ERR_INVALID_PARAMETER)
    with pytest.raises(P.UnsupportedEngine):
        _lib.check(_lib.PRNG_ERR_UNSUPPORTED_ENGINE)
    with pytest.raises(_lib.CudaError):
        _lib.check(_lib.PRNG_ERR_CUDA)


def test_spec_validation_matches_reference():
    import math

    for lo, hi in [(1.0, 1.0), (2.0, -2.0), (0.0, math.inf), (math.nan, 1.0)]:
        with pytest.raises(P.InvalidRange):
            P.Uniform(lo, hi)
    for mean, sd in [(0.0, 0.0), (0.0, -1.0), (math.inf, 1.0), (math.nan, 1.0)]:
        with pytest.raises(P.InvalidParameter):
            P.Gaussian(mean, sd)
    with pytest.raises(P.InvalidParameter):
        P.Uniform(0.0, 1.0, precision="fp16")
    with pytest.raises(P.InvalidParameter):
        P.Lognormal(0.0, 0.0)
    with pytest.raises(P.InvalidParameter):
        P.Gaussian(0.0, 1.0, method="turbo")
    assert P.words_consumed(P.Gaussian(0, 1), 5) == 6
    assert P.words_consumed(P.Lognormal(), 4) == 4
    assert P.words_consumed(P.Uniform(0, 1), 5) == 5


def test_segment_table_chains_positions():
    from paper_2109_01329_b200 import calosim

    tab = calosim.segment_table((1 << 96) + 5, [200000, 3, 7])
    pos = [int(r["pos_lo"]) | int(r["pos_hi"]) << 64 for r in tab]
    assert pos == [(1 << 96) + 5, (1 << 96) + 200005, (1 << 96) + 200008]
    assert tab["out_offset"].tolist() == [0, 200000, 200003]
    assert calosim.allocation(4000) == 200000 and calosim.allocation(70000) == 210000


def test_onemkl_style_engines_track_reference_positions():
    eng = P.Philox4x32x10(777, offset=5)
    assert eng.state == P.skip_ahead(P.seed_engine(P.EngineKind.PHILOX4X32X10, 777), 5)
    eng.skip_ahead(1 << 100)
    assert P.stream_position(eng.state) == 5 + (1 << 100)
    back = P.Philox4x32x10.from_state(eng.state)
    assert back.position == eng.position and back.key == eng.key
    k0, k1, ctr, lane = eng.launch_args()
    blk = eng.position >> 2
    assert list(ctr) == [(blk >> (32 * i)) & 0xFFFFFFFF for i in range(4)] and lane == eng.position & 3
    m = P.Mrg32k3a(4242, offset=1000)
    assert m.state == P.skip_ahead(P.seed_engine(P.EngineKind.MRG32K3A, 4242), 1000)
    with pytest.raises(ValueError):
        m.skip_ahead(-1)
