"""Times the CSR pattern build (k_pattern_rows + k_pattern_cols) of a config:
python tools/time_pattern.py C4"""
import sys
import torch
sys.path.insert(0, ".")
import paper_1905_05417_b200 as lf
from paper_1905_05417_b200 import problem as P

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
prob = P.baseline_config(name)
s = torch.cuda.Stream()
plan = lf.Plan(prob, "fast", 0, stream=s.cuda_stream)
rp = torch.empty(plan.rows + 1, dtype=torch.int64, device="cuda")
cols = torch.empty(plan.nnz, dtype=torch.int32, device="cuda")
plan.build_pattern(rp.data_ptr(), cols.data_ptr())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 10
e0.record(s)
for _ in range(n):
    plan.build_pattern(rp.data_ptr(), cols.data_ptr())
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
b = plan.nnz * 4 + (plan.rows + 1) * 8
print(f"{name} pattern build {ms:.3f} ms, {b / ms / 1e6:.1f} GB/s ({b / 1e9:.2f} GB: int32 cols + int64 row_ptr)")
