"""Seeded input generators (qrng_synth): determinism and shard consistency."""
import numpy as np

import qrng_synth as S


def test_chunked_shards_agree():
    full = S.adc_samples(11, 3 * S.CHUNK + 123, 128, 20)
    for start, count in [(0, 10), (S.CHUNK - 5, 10), (2 * S.CHUNK + 7, S.CHUNK), (5, 3 * S.CHUNK)]:
        assert np.array_equal(S.adc_samples(11, count, 128, 20, start=start), full[start:start + count])


def test_samples_shape_and_moments():
    x = S.adc_samples(2, 1 << 20, 128, 20)
    assert x.dtype == np.uint8
    assert abs(x.mean() - 128) < 0.1 and abs(x.std() - 20) < 0.1


def test_seed_bits_pad_and_determinism():
    a = S.uniform_bits(2, 13925)
    assert a.size == (13925 + 7) // 8
    assert a[-1] & 0x07 == 0  # 13925 = 8*1740 + 5 -> 3 pad bits
    assert np.array_equal(a, S.uniform_bits(2, 13925))
    assert not np.array_equal(a, S.uniform_bits(3, 13925))


def test_workloads_match_baseline_configs():
    assert [(w.n, w.m, w.n_blocks, w.seed_bits) for w in S.CONFIGS.values()] == [
        (1024, 716, 256, 1739), (8192, 5734, 16384, 13925), (65536, 45875, 4096, 111410),
        (1048576, 734003, 256, 1782578)]
    assert all(S.sweep_workload(k).raw_bits == 1 << 30 for k in range(10, 23, 2))
    raw, seed = S.workload_inputs(S.CONFIGS[1], 3, 2)
    assert raw.size == 2 * 1024 // 8 and seed.size == (1739 + 7) // 8
