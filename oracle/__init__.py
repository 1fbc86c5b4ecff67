"""TEST INFRASTRUCTURE ONLY -- parity checkers for the Chimera B200 build.

Nothing under ``oracle/`` is part of the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline / ``--impl reference``
legs may import it, and only as the checker (or the timed reference arm), never
as the thing measured or shipped.

* ``oracle/_ref/libpipesim_ref.so`` -- the unmodified reference library
  (``/root/reference/proj``) compiled in place by ``oracle/Makefile`` plus our
  ``ref_shim.cpp`` C entry points.  Present wherever ``build()`` ran with the
  reference mounted; it travels to the GPU box with the snapshot.
* ``oracle/_build/libtoy_oracle.so`` -- ``toy_oracle.c``, a plain-C fp64
  restatement of the reference ToyModel engine (pinned against ``_ref`` and
  the golden fixtures in ``tests/golden``).
* ``oracle/gpt_oracle.py`` -- numpy restatement of the transformer stage math
  under the reference ``Engine`` semantics (the reference has no transformer:
  pinned by pipelined == sequential SGD and finite differences).
"""
