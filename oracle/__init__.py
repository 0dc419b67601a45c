"""CPU oracle for the joint-acceleration bilateral filter (arXiv 1803.00004, Dai/Yuan/Zhang).

TEST INFRASTRUCTURE ONLY. Nothing in the product path (``paper_1803_00004_b200``, ``include/``,
the CUDA library) may import, call, link or execute anything under ``oracle/``. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs use it.

It is a plain, slow, fp64 numpy implementation of the same N-term approximation the GPU path
computes, written from PAPER.md step by step (line numbers "P:n" refer to
/root/reference/PAPER.md). It shares no code with the CUDA path.

Modules
  fit.py  - range fit (truncated trigonometric basis), 2-D Haar fit
            (P:263-320), best-N selection and the
            Appendix-A lowering of Haar terms to 2-D boxes.
  bf.py   - evaluation: fp64 summed-area tables + the box-filter formula
            eq:numerator_2D_box_N_terms; direct double-loop evaluation of the same
            approximated kernels (pin P1); the dimension-promoted 3-D form (pin P2);
            the brute-force bilateral filter eq:BF.

Readings of the paper (listed in DESIGN.md): the range basis lives on
[-T, T] with T = D (Case 1 substitution), which collapses the z-window;
T_s = r + 1/2 with square truncation; half-open pixel cells; clipped borders; per-k
output factors; den <= 0 falls back to I(x).

Parity status: every function here is pinned by tests in tests/test_oracle_*.py against closed
forms, brute force, invariants and the paper's Table V range row. The Table V *spatial* row
 is not reproducible and is recorded as "parity unpinned"; it pins no
function of this module.
"""
