"""CPU: the chain inputs of the build_system fixtures are reproduced bit for bit (the seeded
random_dtmc generator and the stored reference chains)."""

import pytest

from chain_cases import chain, manifest


@pytest.mark.parametrize("name", sorted(manifest()))
def test_chain_inputs_reproduced(name):
    if manifest()[name]["n"] >= 1_000_000:
        pytest.skip("large chain: covered by the GPU test")
    ch, goals = chain(name)  # asserts the input hashes
    assert ch.n == manifest()[name]["n"] and goals
