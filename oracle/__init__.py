"""CPU oracle for the W4A16 hot path of arXiv 2508.15601 (TurboMind GEMM pipeline).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import anything here.
The product path (`paper_2508_15601_b200`) never imports this package and shares
no code with it: the packed layout, the dequantisation and the GEMM are written
here independently from DESIGN.md §3 (the LAYOUT v1 definition) and §4 (the
numerics readings), which restate PAPER.md §3.1, §3.4 and §4.1.

Modules
  numerics   - software round-to-nearest-even to bf16 / fp16 from float64
  layout_v1  - pack / unpack of u4 codes into LAYOUT v1 (plain index formula)
  quant      - exact fp64 dequantisation and the kernel's declared rounding sequence
  gemm       - C = A . dequant(q, s, z) in fp64 (full or sampled rows)
  compare    - the parity metrics (relative Frobenius error, per-element bound)

Everything is float64 / integer numpy; a library matmul (numpy BLAS, fp64) is the
only library primitive on the GEMM path.  Parity status of each function is
stated in its docstring ("pinned by ..."); none is "parity unpinned".
"""

from . import numerics, layout_v1, quant, gemm, compare  # noqa: F401
