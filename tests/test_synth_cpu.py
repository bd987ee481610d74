"""CPU checks of the seeded input generator (synth/): shard independence (any [start,
start+count) window equals the slice of the whole stream, which multi-GPU sharding relies on), range,
rough uniformity, distinct streams per tensor id, and SplitMix64's published first output."""
import numpy as np

import synth

P62 = 29 * 2**57 + 1
P30 = 998244353


def test_splitmix64_reference_value():
    # SplitMix64 with state 0: first output = mix64(0x9E3779B97F4A7C15) = 0xE220A8397B1DCDAF (published sequence)
    assert int(synth.mix64(np.array([0x9E3779B97F4A7C15], dtype=np.uint64))[0]) == 0xE220A8397B1DCDAF


def test_windows_equal_slices_of_the_stream():
    for p in (P62, P30, 13):
        whole = synth.uniform_mod(7, 3, 0, 5000, p)
        for a, b in ((0, 1), (17, 1000), (4999, 5000), (1234, 4321)):
            assert np.array_equal(synth.uniform_mod(7, 3, a, b - a, p), whole[a:b])
    wb = synth.uniform_bits(7, 4, 0, 3000, 20)
    assert np.array_equal(synth.uniform_bits(7, 4, 1000, 500, 20), wb[1000:1500])


def test_range_and_rough_uniformity():
    for p in (P62, P30):
        x = synth.uniform_mod(1, 0, 0, 200000, p)
        assert x.dtype == np.uint64 and int(x.max()) < p
        # 16 equal bins of [0, p): each within 5% of the expected count
        bins = np.minimum((x.astype(np.float64) / p * 16).astype(np.int64), 15)
        counts = np.bincount(bins, minlength=16)
        assert np.all(np.abs(counts - 200000 / 16) < 0.05 * 200000 / 16), counts
    b = synth.uniform_bits(1, 0, 0, 100000, 20)
    assert int(b.max()) < 2**20 and int(b.min()) >= 0


def test_streams_differ_by_tensor_id_and_seed():
    a = synth.uniform_mod(5, 0, 0, 64, P62)
    assert not np.array_equal(a, synth.uniform_mod(5, 1, 0, 64, P62))
    assert not np.array_equal(a, synth.uniform_mod(6, 0, 0, 64, P62))
    assert synth.config_seed(2) == 0x12052926 ^ 2
