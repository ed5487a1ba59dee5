#!/bin/bash
# Round-2 ncu evidence for the hot pass (run under gpurun; each ncu only
# after the same command exited 0 without it).  The summaries are made on the
# box; only the late-round report is kept (gpurun pulls back <= 64 MiB).
set -x
N="ncu --set full --clock-control none --import-source on"
O=gpurun_out
python scripts/ncu_target.py 3 3 > $O/plain3.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/r02_cfg3_launches.csv python scripts/ncu_target.py 3 3 > $O/ncu_l3.log 2>&1
python scripts/ncu_target.py 3 3 > $O/plain3b.log 2>&1 && \
  timeout 900 $N -k regex:k_pass -s 40 -c 2 -f -o $O/r02_prof_cfg3_kpass python scripts/ncu_target.py 3 3 > $O/ncu_f3.log 2>&1
python scripts/ncu_summary.py $O/r02_prof_cfg3_kpass.ncu-rep > $O/r02_cfg3_ncu_kpass_early.md 2>> $O/ncu_f3.log
rm -f $O/r02_prof_cfg3_kpass.ncu-rep
python scripts/ncu_target.py 4 3 > $O/plain4.log 2>&1 && \
  timeout 900 $N -k regex:k_pass -s 40 -c 1 -f -o $O/r02_prof_cfg4_kpass python scripts/ncu_target.py 4 3 > $O/ncu_f4.log 2>&1
python scripts/ncu_summary.py $O/r02_prof_cfg4_kpass.ncu-rep > $O/r02_cfg4_ncu_kpass.md 2>> $O/ncu_f4.log
rm -f $O/r02_prof_cfg4_kpass.ncu-rep
# late-round capture (round ~90: most coefficients are zero, the axpy of those
# columns is skipped); host loop so that ncu sees every launch
BX_NO_GRAPH=1 python scripts/ncu_target.py 3 100 > $O/plain3c.log 2>&1 && \
  BX_NO_GRAPH=1 timeout 1200 $N -k regex:k_pass -s 950 -c 2 -f -o $O/r02_prof_cfg3_kpass_late python scripts/ncu_target.py 3 100 > $O/ncu_f3c.log 2>&1
python scripts/ncu_summary.py $O/r02_prof_cfg3_kpass_late.ncu-rep > $O/r02_cfg3_ncu_kpass_late.md 2>> $O/ncu_f3c.log
# config 1: the small-round kernel
python scripts/ncu_target.py 1 40 > $O/plain1.log 2>&1 && \
  timeout 900 $N -k regex:k_round_small -c 1 -f -o $O/r02_prof_cfg1_small python scripts/ncu_target.py 1 40 > $O/ncu_f1.log 2>&1
python scripts/ncu_summary.py $O/r02_prof_cfg1_small.ncu-rep > $O/r02_ncu_cfg1_small.md 2>> $O/ncu_f1.log
rm -f $O/r02_prof_cfg1_small.ncu-rep
ls -la $O/
