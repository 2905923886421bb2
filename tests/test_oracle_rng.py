"""Pins for the oracle's counter-based generator and random-init recipe."""
import math

import numpy as np

from oracle.philox import philox4x32_10, stream_words
from oracle import params as OP
from oracle import stages
from synth.configs import TINY, MID

# Random123 known-answer vectors for philox4x32-10 (kat_vectors, Salmon et al. SC'11).
KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


def test_philox_kat():
    for ctr, key, want in KAT:
        out = philox4x32_10(*[np.array([c], dtype=np.uint64) for c in ctr], *key)
        assert tuple(int(o[0]) for o in out) == want


def test_stream_layout():
    # word i is output word (i & 3) of block (i >> 2): check against direct calls
    seed = 0x1234_5678_9ABC_DEF0
    w = stream_words(seed, 11, 7, 0)
    for i in range(11):
        o = philox4x32_10(np.array([i >> 2], np.uint64), np.array([0], np.uint64), np.array([7], np.uint64),
                          np.array([0], np.uint64), seed & 0xFFFFFFFF, seed >> 32)
        assert int(w[i]) == int(o[i & 3][0])


def test_bf16_rne():
    f = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, 1.0 + 2 ** -9, -2.5, 3.0e38], dtype=np.float32)
    bits = OP.f32_to_bf16_rne_bits(f)
    vals = OP.bf16_bits_to_f64(bits)
    # 1+2^-8 is a tie -> even (1.0); 1+3*2^-8 tie -> even (1+2^-6... i.e. 1.015625); 1+2^-9 rounds down
    assert vals[0] == 1.0 and vals[1] == 1.0 and vals[2] == 1.0 + 2 ** -6 and vals[3] == 1.0
    assert vals[4] == -2.5


def test_uniform_recipe_bounds_and_moments():
    cfg = MID
    P = OP.Params(cfg, weight_seed=0)
    w = P["L0.qkv_w"]
    a = math.sqrt(3.0) / math.sqrt(cfg.d)
    assert np.abs(w).max() <= a * (1 + 2 ** -8)
    assert abs(w.mean()) < 3 * (a / math.sqrt(3)) / math.sqrt(w.size)
    assert abs(w.std() / (a / math.sqrt(3)) - 1.0) < 0.01
    g = P["L0.g_q"]
    assert np.all(np.abs(g - 1.0) <= math.sqrt(3) * 0.1 * 1.01)
    # every value is a bf16 number
    bits = P.bits("L0.o_w")
    assert np.array_equal(OP.bf16_bits_to_f64(bits), P["L0.o_w"])


def test_distinct_tensors_distinct_streams():
    P = OP.Params(TINY, 0)
    assert not np.array_equal(P["L0.o_w"], P["L0.co_w"])
    P1 = OP.Params(TINY, 1)
    assert not np.array_equal(P["L0.o_w"], P1["L0.o_w"])


def test_tensor_ids_unique():
    tab = OP.tensor_table(MID)
    ids = [t[0] for t in tab]
    assert len(ids) == len(set(ids))


def test_noise_moments_and_tokens():
    x = stages.noise(MID, seed=5)
    assert x.dtype == np.float32 and x.shape == MID.latent_shape
    assert abs(float(x.mean())) < 0.02 and abs(float(x.std()) - 1.0) < 0.02
    ids = stages.tokens_from_seed(TINY, 3)
    assert ids.min() >= 0 and ids.max() < TINY.vocab and ids.shape == (TINY.L_txt,)


def test_streaming_params_equal_cached_params():
    """tests/oracle_big.StreamingParams (sliced Philox on a pool, no per-layer cache) yields
    the same bf16 bits as oracle.params.Params for every tensor of the mid model."""
    from oracle import params as OP
    from oracle_big import StreamingParams
    from synth.configs import MID
    P, S = OP.Params(MID, 3), StreamingParams(MID, 3, procs=2, slice_words=4096)
    try:
        for _, name, _, _ in OP.tensor_table(MID):
            if name.startswith("L1.") or name.startswith("L0.w") or not name.startswith("L"):
                assert np.array_equal(P.bits(name), S.bits(name)), name
                assert np.array_equal(P[name], S[name]), name
    finally:
        S.close()
