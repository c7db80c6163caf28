"""CPU oracle for the BlockPerm-SJLT sketch apply Y = S·A  (TEST INFRASTRUCTURE ONLY).

This package is a deliberately plain, slow, obviously-correct float64 restatement of
the sketch defined in arXiv 2602.06071 ("FlashSketch"), written from the paper
(`P:n` = line n of /root/reference/PAPER.md) plus the frozen readings recorded in
DESIGN.md §3 for every point the paper leaves open.

Rules (task contract ③):
  * Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
    `--impl reference` legs may import anything from here.  The product path
    (`paper_2602_06071_b200`) never imports, links or executes this package and
    fails loudly when its CUDA library is missing.
  * It shares no code with `paper_2602_06071_b200/csrc` (no headers, helpers,
    constants generators or pre/post-processing).  Inputs come from `synth/`,
    which holds no arithmetic of the method.
  * It builds S explicitly and multiplies — no blocking, fusion or reordering
    beyond the definition.

Pins (what checks the oracle against something other than itself) live in
`tests/test_oracle_*.py`; see DESIGN.md §4 for the pin table.  Functions with no
pin say "parity unpinned" in their docstring (none at present).
"""

from . import blockrow  # noqa: F401  (FlashBlockRow)
from .blockperm import (  # noqa: F401
    MASK64,
    TAG_A,
    TAG_B,
    TAG_PHI,
    Sketch,
    apply,
    apply_adjoint,
    apply_t,
    build_S_csr,
    build_S_dense,
    check_edge_disjoint,
    energy_identity_lhs,
    full_cycle_bruteforce,
    hull_dobell,
    make_sketch,
    mix64,
    neighborhood,
    neighborhoods,
    orbit,
    pattern,
    rad,
    select_affine,
    sketch_rows,
)
