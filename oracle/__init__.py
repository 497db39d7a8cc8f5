"""CPU oracle for the condensed-space ACOPF solve path.

TEST INFRASTRUCTURE ONLY.  Nothing under ``paper_2307_16830_b200/`` may
import, call or link anything in this directory: the oracle is the
checker the GPU path is compared against (tests/, ``__graft_entry__``'s
``smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs), never the thing measured or shipped.

It is a restatement of the reference package ``gridnlp`` 0.1.0
(``/root/reference/pkg/src/gridnlp``): numpy for the vectorised parts and
plain C (``oracle/csrc/chol.c``, built by ``oracle/build.py``) for the two
numba kernels.  Every function cites the reference file:line it follows.

Parity pinning: the oracle is checked against golden vectors produced by
running the reference itself in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz|json``) and
against the known-answer values of the reference's own tests
(``tests/test_oracle_golden.py``).
"""
