"""c1 (axpy + accu, n = 1e6) per-call device time under TMA ring geometry
overrides (COOT_TMA_TILE / COOT_TMA_CTAS / COOT_TMA_SMEM_KB), CUDA-graph
replays as in tools/small_n.py.  usage: python tools/c1_sweep.py"""
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from small_n import mkctx, per_call_us  # noqa: E402

for n in (1_000_000, 4_000_000):
    for tile, ctas, kb in itertools.product((512, 1024, 2048), (1, 2, 3, 4), (32, 64)):
        ctx = mkctx(COOT_TMA_TILE=tile, COOT_TMA_CTAS=ctas, COOT_TMA_SMEM_KB=kb)
        us, grid = per_call_us(ctx, n)
        print(f"n={n} tile={tile} ctas={ctas} kb={kb} grid={grid} {us:.2f} us", flush=True)
