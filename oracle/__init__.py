"""CPU oracle for the B200 engine -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline /
``--impl reference`` leg may import this package.  The product path
(``paper_2101_01332_b200``) never imports it and has no CPU fallback.
"""
