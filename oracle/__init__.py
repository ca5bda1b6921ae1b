"""TEST INFRASTRUCTURE ONLY — the CPU checker for the IVF++ ADSampling path.

Two libraries, same contracts:

* ``liboracle.so``           plain-C restatement of the reference (adsann_oracle.c)
* ``_ref/libadsann_ref.so``  the reference itself, compiled from
                             /root/reference/proj/src by oracle/Makefile

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs may import this package, and only to check or to time the CPU side.
The product package (``paper_2303_09855_b200``) never imports it.
"""
from .oracle import Oracle, RefLib, load_oracle, load_ref, ref_available  # noqa: F401
