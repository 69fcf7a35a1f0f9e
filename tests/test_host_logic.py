"""CPU: host-side logic of the package (seed derivation, WTA parameter
arithmetic) checked against the oracle."""
import pytest

from paper_1806_00588_b200 import bits_for
from paper_1806_00588_b200.seeds import mix_seed


@pytest.mark.parametrize("seed", [0, 1, 7, 2**63 + 5, 123456789])
def test_mix_seed_matches_reference_schedule(oracle, seed):
    for stream in (0, 1, 2, 3, 100, 163):
        assert mix_seed(seed, stream) == oracle.mix_seed(seed, stream)


def test_bits_for():
    assert [bits_for(k) for k in (2, 3, 4, 5, 8, 9, 16, 17)] == [1, 2, 2, 3, 3, 4, 4, 5]
