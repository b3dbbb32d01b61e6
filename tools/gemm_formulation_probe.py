"""The tensor-core alternative for configs[2] inference (north star: "an
int8 tcgen05 0/1-GEMM formulation of the violation count (Include x not-X)
is kept only if ncu shows it beats the LOP3 path").

Violations V[e, r] = sum_p (1 - lit[e, p]) * inc[p, r]; a rule fires iff
V == 0 (and it has includes).  The literals are [x, 1 - x], so
V = sum_f (1 - x_f) inc_pos[f, r] + sum_f x_f inc_neg[f, r]  -- one int8
GEMM of [examples x 2F] by [2F x R].  This probe times that GEMM with the
library int8 path (torch._int_mm -> cuBLASLt, tensor cores) on configs[2]
shapes, checks the formulation against the LOP3 kernel's votes on a sample,
and projects the time for 2^22 examples.  It is a measurement tool, not a
product path."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2405_04212_b200 as tmb  # noqa: E402
from paper_2405_04212_b200 import datasets  # noqa: E402

F, C, K = 4096, 10000, 10
m = datasets.inference_model(model_seed=11)
inc = torch.from_numpy((m.states >= 0).astype(np.int8)).cuda()      # [C, 2F]
w = torch.from_numpy(m.weights.astype(np.int32)).cuda()             # [C, K]
R = ((C + 7) // 8) * 8
incT = torch.zeros((2 * F, R), dtype=torch.int8, device="cuda")
incT[:, :C] = inc.t()
n_inc = inc.sum(dim=1, dtype=torch.int32)
M = 8192
x = bench.c3_inputs_device(M, 0)                                      # uint8 0/1
notlit = torch.cat([1 - x, x], dim=1).to(torch.int8)                  # 1 - literal
viol = torch._int_mm(notlit, incT)[:, :C]                             # [M, C] int32
fire = ((viol == 0) & (n_inc > 0)).to(torch.int32)
votes = fire.to(torch.float64) @ w.to(torch.float64)                  # exact (small ints)
bank = tmb.DenseClauseBank(tmb.Config(n_literals=F, n_clauses=C, n_classes=K, s=2.0,
                                      threshold=100))
bank.states[:] = m.states
bank.weights[:] = m.weights
model = tmb.CompiledModel.from_bank(bank)
v_lop3, _ = model.votes_and_pred(x.cpu().numpy())
same = bool(np.array_equal(votes.round().long().cpu().numpy(), v_lop3))
# throughput of the violation GEMM alone (the second GEMM is K=10 wide)
for _ in range(3):
    torch._int_mm(notlit, incT)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 10
a.record()
for _ in range(reps):
    torch._int_mm(notlit, incT)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
ops = 2.0 * M * (2 * F) * R
print(f"int8 GEMM [{M} x {2 * F}] x [{2 * F} x {R}]: {ms:.3f} ms, {ops / ms / 1e9:.1f} TOP/s")
print(f"projected violation GEMM for 2^22 examples: {ms * (1 << 22) / M:.1f} ms "
      f"(LOP3 path k_infer_ws: ~7.9 ms for the whole inference)")
print(f"GEMM formulation votes == LOP3 kernel votes on {M} examples: {same}")
