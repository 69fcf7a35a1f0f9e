"""SplitMix64 seed derivation (include/lshbeam/rng.hpp:15-20, :49-52), used to
derive the WTA / cuckoo seeds from one model seed the way the reference CLI
does (tools/main.cpp:81-82: perm seed mix_seed(seed,1), index seed
mix_seed(seed,2))."""

M64 = (1 << 64) - 1


def splitmix_next(state: int):
    state = (state + 0x9E3779B97F4A7C15) & M64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31), state


def mix_seed(seed: int, stream: int) -> int:
    s = (seed ^ ((0xBF58476D1CE4E5B9 * (stream + 1)) & M64)) & M64
    return splitmix_next(s)[0]
