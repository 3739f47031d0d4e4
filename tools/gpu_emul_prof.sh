#!/bin/bash
mkdir -p gpurun_out
cat > /tmp/emul1.py <<'PY'
import os, sys
os.environ["MSTRSM_DIST_EMULATE_P"] = "8"; os.environ["MSTRSM_DIST_TEST_UNPACK"] = "1"
sys.path.insert(0, os.getcwd())
import torch
import paper_1607_01477_b200 as ms
from paper_1607_01477_b200 import inputs
ms.load()
T = torch.from_numpy(inputs.c5_grcar_like(16384)).cuda()
ms.comm_init(1, 0)
ms.trevc_dist(T, 16384, nb=128); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
ms.trevc_dist(T, 16384, nb=128); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
PY
python /tmp/emul1.py > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --profile-from-start off \
  --log-file gpurun_out/launch_emul_r02.csv python /tmp/emul1.py > /dev/null 2>&1
echo $?
