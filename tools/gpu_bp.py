#!/usr/bin/env python
"""BP3 / BP4 / BP5 of the reference's harness (bench.py:153-212 defaults) on the B200 through harness.bench_csv:
the frozen `mfcg bench` CSV, min of 3 repeats of 50 fixed iterations."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2205_08909_b200 import harness
from paper_2205_08909_b200.mesh import GeometryVariant

rows = []
for bp, p, n, kw in [("BP5", 5, 58, {}), ("BP3", 5, 40, {}), ("BP4", 5, 28, {}),
                     ("BP4", 5, 40, dict(geometry=GeometryVariant.AFFINE, deform=0.0))]:
    for variant in ("pcg", "combined_pcg"):
        rec = harness.run_benchmark(bp, p, (n, n, n), variant, iterations=50, repeats=3, **kw)
        rows.append(rec)
        print(bp, p, n, variant, kw, f"{rec.throughput:.3e} DoF*it/s", flush=True)
out = Path(__file__).resolve().parent.parent / "gpurun_out" / "r02_bp.csv"
out.parent.mkdir(exist_ok=True)
print(harness.write_bench_csv(rows, out))
