#!/bin/bash
# Round-2 (late) profiling pass of the final code (ONE GPU, under gpurun).  Outputs in gpurun_out/.
#  1. launch list of the default bench command (LLaMA-7B Adam headline), single-pass metric;
#     application replay so ncu never saves/restores the 94 GB working set
#  2. DRAM traffic of the headline's step-kernel launch (application replay, 1 pass)
#  3. ncu --set full of the step kernel on the Adam / SGD / clip workloads (kernel replay)
#  4. ncu --set full of the fused P2P sharded step (bulk-copy pipeline) at world 1
set -x
B="python bench.py --steps 20 --warmup 5 --no-secondary --no-cpu-baseline --e2e-steps 3"
timeout 900 ncu --replay-mode application --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_llama7b_adam.csv $B > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --replay-mode application --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:step_tma -s 8 -c 1 -o gpurun_out/prof_llama7b_adam \
    python bench.py --steps 8 --warmup 5 --no-secondary --no-cpu-baseline --e2e-steps 3 > gpurun_out/ncu_llama.log 2>&1
for w in gpt2_adamw resnet50_sgd vit_l16_adam_clip; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"step_tma|sumsq" -s 12 -c 3 \
      -o gpurun_out/prof_$w python bench.py --workload $w --steps 12 --warmup 3 --no-secondary --no-cpu-baseline --e2e-steps 3 \
      > gpurun_out/ncu_full_$w.log 2>&1
done
cat > /tmp/p2p_one.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2309_12381_b200 as mpo
from paper_2309_12381_b200 import api
from paper_2309_12381_b200._lib import MPO_ADAM
n = 124439808 // 8 * 8
V = (torch.randn(n, device="cuda") * 0.02).to(torch.bfloat16)
G = (torch.randn(n, device="cuda") * 1e-3).to(torch.bfloat16)
R = torch.zeros(n, dtype=torch.int16, device="cuda"); M = torch.zeros(n, device="cuda"); W = torch.zeros(n, device="cuda")
hp = mpo.AdamParams(lr=1e-3)
for _ in range(4):
    api.mpo_p2p_sharded_step(MPO_ADAM, 0, 1, [V.data_ptr()], [G.data_ptr()], R, M, W, n, hp, torch.bfloat16)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:p2p -s 2 -c 1 \
    -o gpurun_out/prof_p2p_gpt2_world1 python /tmp/p2p_one.py > gpurun_out/ncu_p2p.log 2>&1
# 5. the NVLS kernel with emulated multicast (2 ranks on one device, GPT-2-sized flat buffer)
cat > /tmp/nvls_emu.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2309_12381_b200 as mpo
from paper_2309_12381_b200 import api
from paper_2309_12381_b200._lib import MPO_ADAM
W = 2
n = 124439808 // 16 * 16
S = n // W
V = [(torch.randn(n, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(W)]
G = [(torch.randn(n, device="cuda") * 1e-3).to(torch.bfloat16) for _ in range(W)]
st = [(torch.zeros(S, dtype=torch.int16, device="cuda"), torch.zeros(S, device="cuda"), torch.zeros(S, device="cuda"))
      for _ in range(W)]
hp = mpo.AdamParams(lr=1e-3, grad_scale=0.5)
for _ in range(3):
    for k in range(W):
        api.mpo_nvls_emulated_step(MPO_ADAM, k, W, [t.data_ptr() for t in V], [t.data_ptr() for t in G], *st[k], n, hp,
                                   torch.bfloat16)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nvls -s 2 -c 1 \
    -o gpurun_out/prof_nvls_emulated_gpt2_world2 python /tmp/nvls_emu.py > gpurun_out/ncu_nvls.log 2>&1
ls -la gpurun_out/*.ncu-rep
