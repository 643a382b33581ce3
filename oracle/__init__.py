"""ORACLE -- test infrastructure, never the product.

CPU restatements the B200 build is checked against:

* ``hashinit``  -- the counter-based synthetic init (weights, prompt ids);
* ``decoder``   -- the per-stage decoder forward (bf16-faithful torch CPU),
  the computation the reference replaces with ``compute_time``
  (pipelink/engine.py:384);
* the scheduling / chunking / link-timing half of the path is the reference
  itself: ``pipelink`` imported unmodified (``PipelineEngine.run`` is the
  schedule oracle; ``LinkQueue``/``replay_link`` the chunk oracle).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package.
"""
