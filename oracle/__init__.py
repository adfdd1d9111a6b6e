"""CPU oracle for the SubApSnap online phase — TEST INFRASTRUCTURE ONLY.

A plain numpy/scipy restatement of the reference's online path
(/root/reference/pkg/src/subapsnap/online.py, linalg.py) used as the checker
for the CUDA path.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import it; the product path
(paper_2510_04825_b200) never does.

Pinned against the reference itself: tests/golden/*.npz were produced by
running the unmodified reference package (PYTHONPATH=/root/reference/pkg/src)
with tests/golden/make_golden.py, and tests/test_oracle_golden.py checks this
restatement against them.
"""
