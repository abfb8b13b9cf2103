"""CPU oracle for the IRL-SR hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU reference — never as the product path (which runs exclusively
in ``libirlsr.so`` on sm_100a and fails loudly without it).

Contents (numpy restatements; every function cites the reference file:line):

* ``estimators`` — est:146-186, est:319-344 (energy, gradient, centred products)
* ``krylov``     — kry:87-345 (Lanczos, implicit restart, IRL k=1)
* ``bordered``   — opt:138-165 (bordered closure, update direction)
* ``nqs``        — RBM / MLP rows and log psi (no reference function: pinned by
                   central finite differences, T/test_ansatz.py:67-81 pattern,
                   and by the reference phase-head gradient, ans:278-288)

Pinning: ``make_golden.py`` imports the real reference (``/root/reference``,
this container only) and writes ``tests/golden/*.npz``; the CPU tests check
this restatement against those vectors.
"""
