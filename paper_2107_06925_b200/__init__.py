"""Chimera bidirectional pipeline training, B200-native (sm_100a).

Layers:
  * ``pipesim``  -- Python mirror of the reference schedule API (C++ host layer).
  * ``toy``      -- the reference ToyModel executed by sm_100a kernels (parity path).
  * ``gpt``      -- GPT-2 stage-partitioned training under a Chimera schedule.
All compute goes through libchimera.so (include/chimera_ck.h); there is no CPU
fallback.
"""
__all__ = ["pipesim"]
