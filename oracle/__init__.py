"""CPU oracle for the OmniSparse sparse-attention hot path — TEST INFRASTRUCTURE ONLY.

This package is a float64 NumPy restatement of the reference package
``slimattn`` (``/root/reference/pkg/src/slimattn``); every function cites the
reference file:line it follows. It exists to CHECK the CUDA path:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import it;
* the product package ``paper_2511_12201_b200`` never imports it and has no
  CPU fallback — its ops fail loudly when the CUDA library is missing.

Parity pinning: ``tests/golden/make_golden.py`` runs the reference itself (in
the build container, where ``/root/reference`` exists) and commits its outputs
as fixtures; ``tests/test_oracle_golden.py`` checks this restatement against
them. GQA (28 Q / 4 KV heads) is outside the reference (``SPEC.md:145``); the
rule-B composition in :mod:`oracle.pipeline` is built only from restated
reference functions and reduces exactly to the reference at Hq == Hkv (pinned
by the same fixtures). Gradients have no reference (no autograd anywhere in
``slimattn``): :mod:`oracle.grad` is a float64 torch-autograd restatement whose
forward is pinned to ``sparse_head_attention`` — "parity pinned for forward,
gradient oracle derived".
"""
