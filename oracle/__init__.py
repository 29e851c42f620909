"""CPU oracle for the bpqn hot path (arXiv 2604.10089) -- TEST INFRASTRUCTURE ONLY.

This package is a plain, slow, obviously-correct fp64 CPU implementation of the
discretised LCP matrix-vector product w = D^T M D lambda and of
the paper's Mono-PQN / Bi-PQN solvers (Alg. 1, Alg. 2 P:372-388,
Alg. 3, Alg. 4).  Where the paper is silent (the whole Stokes
boundary-integral discretisation, P:425-426 only names it) the oracle follows the
readings R1..R30 frozen in DESIGN.md / SURVEY.md section 8(c).

Rules:
  * Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
    ``--impl reference`` legs may import or execute anything under ``oracle/``.
  * The oracle shares no code with the CUDA path (``paper_2604_10089_b200/``);
    neither imports the other.  Only the seeded input generators in ``synth/``
    (which hold none of the method's arithmetic) serve both.

Parity status per function is listed in each module header; every function is
pinned by a ``-m "not gpu"`` test in ``tests/test_oracle_*.py`` unless its header
says "parity unpinned".
"""
