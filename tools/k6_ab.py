"""Times the standard (full 3D quadrature, K6) assembly of a BASELINE config
and checks it against the fast assembly on the device (both plans share the
closed-form pattern, so their value arrays align entry by entry):
  LAMFAST_LIB=build/k6v/<variant>/liblamfast_b200.so python tools/k6_ab.py C3 [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1905_05417_b200 as lf  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
prob = lf.baseline_config(name)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
std = lf.Plan(prob, "standard", 0, stream=s.cuda_stream)
fast = lf.Plan(prob, "fast", 0, stream=s.cuda_stream)
vs = torch.empty(std.nnz, dtype=torch.float64, device="cuda")
vf = torch.empty(fast.nnz, dtype=torch.float64, device="cuda")
fast.assemble(vf.data_ptr())
std.assemble(vs.data_ptr())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(steps):
    std.assemble(vs.data_ptr())
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
rel = float(torch.linalg.vector_norm(vs - vf) / torch.linalg.vector_norm(vf))
print(f"{name} standard {ms:.2f} ms/step ({std.nnz / ms / 1e6:.3e} nnz/s, launches/step={std.launch_count}), "
      f"||std - fast|| / ||fast|| = {rel:.2e}  lib={os.environ.get('LAMFAST_LIB', 'default')}")
