"""Out-of-bounds checks without a sanitizer (compute-sanitizer is closed on
this GPU pool): every kernel path runs on operands framed by guard bands.

  * inputs sit inside NaN bands — a read past either end turns the result
    non-finite;
  * outputs sit inside bands of a sentinel bit pattern — a write past either
    end changes a sentinel;
at 32-byte-aligned and misaligned offsets, for shapes that select each kernel
(the same list as tools/sanitize_driver.py).  Reruns under
CABL_GEMV_RM_ORDER=reference from the reference-order subprocess test.
"""
from __future__ import annotations

import pytest
import torch

pytestmark = pytest.mark.gpu

PAD = 4096
SENTINEL = 1234.5678


def framed_input(n, dtype, stream, off, cuda):
    import paper_2108_02025_b200 as cb
    big = torch.full((PAD + off + n + PAD,), float("nan"), dtype=dtype, device=cuda)
    if n:
        big[PAD + off:PAD + off + n] = cb.fill_uniform(torch.empty(n, dtype=dtype, device=cuda),
                                                       11, stream)
    return big[PAD + off:PAD + off + n]


class FramedOutput:
    def __init__(self, n, dtype, stream, off, cuda):
        import paper_2108_02025_b200 as cb
        self.big = torch.full((PAD + off + n + PAD,), SENTINEL, dtype=dtype, device=cuda)
        self.lo, self.hi = PAD + off, PAD + off + n
        if n:
            self.big[self.lo:self.hi] = cb.fill_uniform(torch.empty(n, dtype=dtype, device=cuda),
                                                        11, stream)
        self.view = self.big[self.lo:self.hi]

    def check(self, what):
        torch.cuda.synchronize()
        assert bool((self.big[:self.lo] == SENTINEL).all()), f"{what}: write before the output"
        assert bool((self.big[self.hi:] == SENTINEL).all()), f"{what}: write after the output"
        assert bool(torch.isfinite(self.view).all()), f"{what}: read outside an input"


DTYPES = [torch.float32, torch.float64]
OFFSETS = [0, 1]  # elements: 32-byte aligned (PAD*s is), and misaligned


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("off", OFFSETS)
def test_dot_guard_bands(cuda, dtype, off):
    import paper_2108_02025_b200 as cb
    pol = cb.default_policy(1)
    for n in (0, 5, 8192, 8193, 100_003, 1 << 20):
        x, y = framed_input(n, dtype, 1, off, cuda), framed_input(n, dtype, 2, 3 * off, cuda)
        out = FramedOutput(1, dtype, 9, off, cuda)
        cb.dot_into(x, y, 0.5, out.view, pol)
        out.check(f"dot n={n} off={off}")


RM = [(3, 5), (40, 1024), (2, 65536), (7200, 256), (3000, 999), (5000, 1028), (4736, 100),
      (20_000, 16), (20_000, 256), (20_000, 33), (9000, 8200), (1, 1 << 18), (5, 40_000),
      (700, 5003),
      # the sub-CTA sweep: partly filled 128- / 16- / 32-lane row slots, ragged last group
      (9473, 520), (10_001, 72), (9999, 1000), (9601, 144), (9473, 1288), (9500, 2048),
      # the scalar sub-CTA sweep (odd rows; with an offset every shape here is scalar too)
      (9473, 65), (9601, 1001), (9500, 2047), (10_000, 130)]
CM = [(3, 5), (256, 4096), (4096, 300), (2008, 77), (1001, 300), (148 * 256 * 8, 4),
      (148 * 1024 + 1, 3), (1, 100_000), (257, 20_000), (74 * 256 * 8, 20), (8193, 300),
      (1025, 777), (3001, 129), (4096, 100), (8192, 301), (512, 5000), (1000, 3)]


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("off", OFFSETS)
@pytest.mark.parametrize("layout", ["row", "col"])
def test_gemv_guard_bands(cuda, dtype, off, layout):
    import paper_2108_02025_b200 as cb
    pol = cb.default_policy(1)
    lay = cb.Layout.RowMajor if layout == "row" else cb.Layout.ColMajor
    f = cb.gemv_row_major if layout == "row" else cb.gemv_col_major
    for m, n in (RM if layout == "row" else CM):
        A = framed_input(m * n, dtype, 3, off, cuda)
        x = framed_input(n, dtype, 1, off, cuda)
        c = FramedOutput(m, dtype, 4, off, cuda)
        f(cb.DenseMatrix.wrap(A, m, n, lay), x, c.view, pol)
        c.check(f"gemv {layout} {m}x{n} off={off}")


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("off", OFFSETS)
@pytest.mark.parametrize("layout", ["row", "col"])
def test_ger_guard_bands(cuda, dtype, off, layout):
    import paper_2108_02025_b200 as cb
    pol = cb.default_policy(1)
    lay = cb.Layout.RowMajor if layout == "row" else cb.Layout.ColMajor
    for m, n in ((3, 5), (37, 1000), (300, 2048), (1000, 4096), (8, 8193), (20_000, 64),
                 (3000, 4100), (50_000, 5), (777, 1001), (1001, 777), (400, 1003),
                 (400_003, 1), (1, 400_003)):
        x, y = framed_input(m, dtype, 1, off, cuda), framed_input(n, dtype, 2, off, cuda)
        C = FramedOutput(m * n, dtype, 5, off, cuda)
        cb.ger(x, y, cb.DenseMatrix.wrap(C.view, m, n, lay), pol)
        C.check(f"ger {layout} {m}x{n} off={off}")
