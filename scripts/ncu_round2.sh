#!/bin/bash
# Round-2 ncu evidence for the hot pass (run under gpurun; each ncu only
# after the same command exited 0 without it).
set -x
N="ncu --set full --clock-control none --import-source on"
python scripts/ncu_target.py 3 3 > gpurun_out/plain3.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02_cfg3_launches.csv python scripts/ncu_target.py 3 3 > gpurun_out/ncu_l3.log 2>&1
python scripts/ncu_target.py 3 3 > gpurun_out/plain3b.log 2>&1 && \
  timeout 900 $N -k regex:k_pass -s 40 -c 2 -f -o gpurun_out/r02_prof_cfg3_kpass python scripts/ncu_target.py 3 3 > gpurun_out/ncu_f3.log 2>&1
python scripts/ncu_target.py 4 3 > gpurun_out/plain4.log 2>&1 && \
  timeout 900 $N -k regex:k_pass -s 40 -c 1 -f -o gpurun_out/r02_prof_cfg4_kpass python scripts/ncu_target.py 4 3 > gpurun_out/ncu_f4.log 2>&1
ls -la gpurun_out/
# late-round capture (round ~90: most coefficients are zero, the axpy of those
# columns is skipped); host loop so that ncu sees every launch
BX_NO_GRAPH=1 python scripts/ncu_target.py 3 100 > gpurun_out/plain3c.log 2>&1 && \
  BX_NO_GRAPH=1 timeout 1200 $N -k regex:k_pass -s 950 -c 2 -f -o gpurun_out/r02_prof_cfg3_kpass_late python scripts/ncu_target.py 3 100 > gpurun_out/ncu_f3c.log 2>&1
