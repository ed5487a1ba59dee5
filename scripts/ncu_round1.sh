set -x
N="ncu --set full --clock-control none --import-source on"
python scripts/ncu_target.py 4 3 && timeout 600 $N -k regex:k_pass -s 5 -c 1 -f -o gpurun_out/prof_cfg4_kpass python scripts/ncu_target.py 4 3 > gpurun_out/ncu_cfg4.log 2>&1
python scripts/ncu_target.py 1 3 && timeout 600 $N -k regex:k_round_small -c 1 -f -o gpurun_out/prof_cfg1_small python scripts/ncu_target.py 1 3 > gpurun_out/ncu_cfg1.log 2>&1
python scripts/ncu_target.py 2 3 && timeout 600 $N -k regex:k_cd -s 1 -c 1 -f -o gpurun_out/prof_cfg2_cd python scripts/ncu_target.py 2 3 > gpurun_out/ncu_cfg2.log 2>&1
python scripts/ncu_batched.py && timeout 900 $N -k regex:k_batched_round -c 1 -f -o gpurun_out/prof_cfg5_batched python scripts/ncu_batched.py > gpurun_out/ncu_cfg5.log 2>&1
python scripts/ncu_target.py 1 40 active-set && timeout 600 $N -k regex:k_as_solve -s 20 -c 1 -f -o gpurun_out/prof_as_solve python scripts/ncu_target.py 1 40 active-set > gpurun_out/ncu_as.log 2>&1
ls -la gpurun_out/
