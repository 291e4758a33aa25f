#!/bin/bash
# determinism probe: four applies of one plan compared bit for bit -- the default launch modes against
# owned items (FDA_GT_MODE=owned: plain read-modify-write, no FP64 reductions) + one-sided P2P, with the
# warp-task M2L, without it, and with the two-pass block M2L (FDA_M2L_BLOCK=1); CONFIGS="1b 3" by default
mkdir -p gpurun_out
for c in ${CONFIGS:-1b 3}; do
  TAG=a timeout 600 python tools/det_probe.py $c >> gpurun_out/det.log 2>&1
  TAG=b FDA_GT_MODE=owned FDA_P2P_SYM=0 timeout 600 python tools/det_probe.py $c >> gpurun_out/det.log 2>&1
  TAG=c FDA_GT_MODE=owned FDA_P2P_SYM=0 FDA_M2L_BLOCK=1 timeout 600 python tools/det_probe.py $c >> gpurun_out/det.log 2>&1
  python -c "
import numpy as np
a=np.load('/tmp/det_a.npy');b=np.load('/tmp/det_b.npy');c=np.load('/tmp/det_c.npy')
print('rel b-a', np.linalg.norm(b-a)/np.linalg.norm(a), 'rel c-a', np.linalg.norm(c-a)/np.linalg.norm(a))" >> gpurun_out/det.log 2>&1
done
