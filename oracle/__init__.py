"""CPU oracle for the GO (arXiv 2010.12438) policy-evaluation path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2010_12438_b200`` imports this
package; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may use it, and only as the
checker (or the timed CPU baseline), never as the thing measured or shipped.

It is a float64 numpy / pure-Python restatement of the reference package
``graphopt`` (``/root/reference/pkg/src/graphopt``); every function cites the
reference file:line it follows.  Parity is pinned by ``tests/golden/*.npz``,
generated from the unmodified reference by ``tests/golden/make_golden.py``
(see ``tests/test_oracle_golden.py``).
"""
