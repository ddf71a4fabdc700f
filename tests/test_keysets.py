"""Key sets of BASELINE.json's configs: the frozen
torchvision parameter sizes and the pinned C5 stress generator.  CPU only."""
import _oracle as O

from paper_1802_06949_b200 import keysets


def test_frozen_model_key_sets_match_the_survey():
    expect = {"resnet50": (161, 25_557_032), "alexnet": (16, 61_100_840), "resnet152": (467, 60_192_808),
              "inception_v3": (292, 27_161_264)}
    for name, (k, total) in expect.items():
        sizes = keysets.load(name)
        assert (len(sizes), sum(sizes)) == (k, total), name
    assert keysets.load("uniform16x1048576") == [1 << 20] * 16


def test_stress_generator_is_the_reference_mt19937_64():
    # u = top 53 bits of std::mt19937_64(0), the same draw random_uniform maps to [-1, 1)
    g = keysets._mt19937_64(0)
    u = (next(g) >> 11) * 2.0 ** -53
    assert u * 2.0 - 1.0 == O.random_uniform(1, 0)[0]
    sizes = keysets.stress_keys()
    nbytes = [4 * n for n in sizes]
    assert len(sizes) == 2048
    assert min(nbytes) >= 1024 and max(nbytes) <= 64 << 20
    assert 10 << 30 < sum(nbytes) < 14 << 30  # ~12 GiB per GPU
    assert keysets.stress_keys(96) == sizes[:96]
