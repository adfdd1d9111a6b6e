"""CPU oracle for the SubApSnap online phase — TEST INFRASTRUCTURE ONLY.

A plain numpy/scipy restatement of the reference's online path
(/root/reference/pkg/src/subapsnap/online.py, linalg.py) used as the checker
for the CUDA path.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import it; the product path
(paper_2510_04825_b200) never does.

The arithmetic the reference delegates to third-party code is not vendored in
/root/reference: pyproject.toml:10-15 pins only lower bounds, so the de facto
pins are this image's numpy 2.3.5 (linalg.qr -> LAPACK dgeqrf/dorgqr, zgeqrf/
zungqr via OpenBLAS 0.3.30), scipy 1.18.1 (linalg.solve_triangular -> dtrtrs,
scipy.sparse CSR products) and numba 0.65.0 (the 1-D rbf_rows kernel); the
restatement calls the same routines (Householder QR, triangular solve).

Pinned against the reference itself: tests/golden/*.npz were produced by
running the unmodified reference package (PYTHONPATH=/root/reference/pkg/src)
with tests/golden/make_golden.py, and tests/test_oracle_golden.py checks this
restatement against them.
"""
