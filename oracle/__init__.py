"""CPU oracle for the AZ step-1 hot path of arXiv:2308.14490.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import anything in
this package.  The product path (paper_2308_14490_b200/, libaz.so) never
imports, links or executes it, and this package never imports the product's
binding or CUDA code: the only shared module is the seeded input generator
`paper_2308_14490_b200.inputs`, which holds no method arithmetic.

Every function is plain, slow and written to be checked against the paper by
eye.  Citations are PAPER.md line numbers (section / equation / algorithm).

Modules
  kernel     Gaussian RBF, its second derivative, periodisation, Eq. (4)
  circulant  block-column circulant structure: Pi, F, P, B, B^dagger, Z* (Sec. 3.1, 5.1, 6.2.2)
  dense      dense collocation matrices A, A^c, boundary rows (Sec. 2.3, 5.2, 6.2.1)
  az         Alg. 1 (dense and FFT-operator versions), truncated-SVD LSQ, evaluation
  philox     Philox4x32-10 + Box-Muller probe generator (independent implementation)

Parity status of each function is listed in DESIGN.md ("Oracle pins").  No
function in this package is "parity unpinned".
"""
