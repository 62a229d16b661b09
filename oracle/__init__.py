"""CPU oracle for the AttentionStore KV-reuse prefill path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2403_19708_b200`` imports this
package; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may use it, and only as the
checker (never as the thing measured or shipped).

The reference (``kvsim`` 0.1.0, /root/reference/pkg/src/kvsim) is pure Python
on numpy, so the oracle is a numpy float64 restatement of the functions on the
hot path.  Every function cites the reference file:line it follows.  The
restatement is *pinned* against golden vectors produced by running the
reference itself in the build container (``tests/golden/make_golden.py``,
fixtures committed under ``tests/golden/``); ``tests/test_oracle_golden.py``
checks it.

Modules
-------
rope_ref      decoupled-PE attention numerics (rope.py)
layout_ref    truncation / block accounting arithmetic (sim.py, store.py, model.py)
overlap_ref   analytical pre-load / async-save timelines (overlap.py)
llama_ref     float64 LLaMA-shaped forward with KV reuse (config C1)
workload_ref  per-turn shapes replayed from committed session fixtures
"""
