"""CPU ORACLE for CBC (arXiv 2601.19650) — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct NumPy (complex128 / fp64) following PAPER.md §III step by
step.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import this package.  The product path
(`paper_2601_19650_b200/`) never imports it and shares no code with it; the two meet
only in the seeded input generators of `workloads/` (which hold no method arithmetic).

Modules
  ttn     containers, dense brute force (Eq. 2 / Eq. 4), overlap / norm sweeps,
          exact (uncompressed) O|psi>
  cbc     tree CBC, Eqs. 10-14 + assembly
  cbc_tt  tensor-train CBC, Eqs. 5-9
  direct  contract-then-truncated-SVD sweep (cross-check, P10)

Pinned by tests/test_oracle_*.py (pins P1-P13 of DESIGN.md §4).  Parity unpinned:
the VALUES of truncated results at config 2-5 sizes (only invariants P2, P3, P4, P7,
P13 hold there) — see DESIGN.md §4.
"""
from .ttn import TTN, to_dense_state, to_dense_operator, overlap, norm, exact_apply, sandwich
from .cbc import cbc_apply, svd_compress, gram_compress, qr_pos, phi
from .cbc_tt import cbc_apply_tt
from .direct import direct_apply

__all__ = ["TTN", "to_dense_state", "to_dense_operator", "overlap", "norm", "exact_apply", "sandwich",
           "cbc_apply", "svd_compress", "gram_compress", "qr_pos", "phi", "cbc_apply_tt", "direct_apply"]
