"""Host side of the random streams (rng.py:19-56 of the reference).

Only the per-worker stream seeding lives on the host; every draw is made on
the device (splitmix64 batches of 32 per warp, or Philox4x32-10 counters).
"""

GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
MASK = 0xFFFFFFFFFFFFFFFF


def _mix(z: int) -> int:
    z &= MASK
    z = ((z ^ (z >> 30)) * MIX1) & MASK
    z = ((z ^ (z >> 27)) * MIX2) & MASK
    return z ^ (z >> 31)


def new_state(seed: int, stream: int = 0) -> int:
    """Initial splitmix64 state of stream (seed, stream), as rng.new_state."""
    return _mix((seed & MASK) ^ ((stream * GOLDEN + 1) & MASK))
