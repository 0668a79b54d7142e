"""CPU oracle for the BTA hot path — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference's algorithms (stinla, pure Python on
numpy/scipy, mounted read-only at /root/reference during development), each
function citing the reference file:line it follows.  It is imported only by
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs, always as the checker or the timed CPU baseline,
never as the product path: the package ``paper_2507_06938_b200`` never imports
it and has no CPU fallback.

Pinning: the restatement is checked against golden vectors produced by the
unmodified reference (``oracle/make_golden.py`` → ``tests/golden/*.npz``) and
against the reference tests' closed-form known answers
(``tests/test_oracle_golden.py``).
"""
