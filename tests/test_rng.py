"""CPU: the C oracle of the reference's random streams (oracle/strait_rng_oracle.c)
equals numpy 2.3 itself — SeedSequence states, PCG64 raw output, ziggurat
exponential / normal draws (tails included) and gen_poisson arrival streams —
so it can pin the device generator (tests/test_rng_gpu.py)."""
import ctypes as C

import numpy as np
import pytest


def _lib(oracle):
    lib = oracle.lib()
    vp = C.c_void_p
    lib.oracle_seedseq_state.argtypes = [vp, C.c_int, vp]
    lib.oracle_rng_raw.argtypes = [vp, C.c_int, C.c_int64, vp]
    lib.oracle_rng_draws.argtypes = [vp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int64, vp]
    lib.oracle_gen_poisson.argtypes = [vp, C.c_int, C.c_double, C.c_double, vp, C.c_int64]
    lib.oracle_gen_poisson.restype = C.c_int64
    return lib


ENTROPIES = ([0, 0], [1, 3], [123456, 5], [2 ** 40 + 7, 2], [3, 1, 17], [7, 1_000_003])


@pytest.mark.parametrize("ent", ENTROPIES)
def test_seedsequence_and_pcg64(oracle, ent):
    lib = _lib(oracle)
    e = np.array(ent, dtype=np.uint64)
    st = np.zeros(4, np.uint64)
    lib.oracle_seedseq_state(e.ctypes.data, len(e), st.ctypes.data)
    np.testing.assert_array_equal(st, np.random.SeedSequence(ent).generate_state(4, np.uint64))
    raw = np.zeros(500, np.uint64)
    lib.oracle_rng_raw(e.ctypes.data, len(e), 500, raw.ctypes.data)
    np.testing.assert_array_equal(raw, np.random.default_rng(np.random.SeedSequence(ent)).bit_generator.random_raw(500))


@pytest.mark.parametrize("ent", ENTROPIES[:3])
def test_ziggurat_draws(oracle, ent):
    lib = _lib(oracle)
    e = np.array(ent, dtype=np.uint64)
    n = 400_000
    for kind, want in ((0, np.random.default_rng(np.random.SeedSequence(ent)).exponential(2.5, n)),
                       (1, np.random.default_rng(np.random.SeedSequence(ent)).normal(0.0, 0.05, n))):
        got = np.zeros(n)
        lib.oracle_rng_draws(e.ctypes.data, len(e), kind, 0.0, 2.5 if kind == 0 else 0.05, n, got.ctypes.data)
        np.testing.assert_array_equal(got, want)


def test_gen_poisson(oracle):
    from paper_2604_28175_b200.workload import gen_poisson_array

    lib = _lib(oracle)
    for ent, rate, dur in (([4, 0], 2200.0, 3000.0), ([9, 5], 3.5, 60000.0), ([1, 2, 7], 2500.0, 1234.5)):
        want = gen_poisson_array(rate, dur, np.random.SeedSequence(ent))
        e = np.array(ent, dtype=np.uint64)
        got = np.zeros(len(want) + 8)
        n = lib.oracle_gen_poisson(e.ctypes.data, len(e), rate, dur, got.ctypes.data, len(got))
        assert n == len(want)
        np.testing.assert_array_equal(got[:n], want)
