"""CPU oracle for the EDPC hot path -- TEST INFRASTRUCTURE, NOT PRODUCT.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package, and only
as the checker / the timed CPU baseline.  The product package
(``paper_2507_18969_b200``) never imports it and has no CPU fallback.

Contents:
* ``edpc_oracle.c`` -- C restatement of the reference's numba kernels
  (quantizer, arithmetic coder, Adam, GeLU), built by ``build.sh``;
* ``coder.py``      -- ctypes wrapper with the reference's coder API;
* ``model.py``      -- numpy float64 restatement of nn.py + model.py;
* ``pipeline.py``   -- serial compress/decompress over the two;
* ``make_goldens.py`` -- regenerates ``tests/golden/`` from the reference
  itself (needs ``/root/reference``; run in the dev container only).

Parity is pinned: tests/test_oracle_golden.py checks this oracle against the
golden vectors the reference produced (bit-exact for the coder, quantizer and
the whole container).
"""
