#!/bin/bash
# last GPU round of round 2: ncu --set full captures of the rank-16 classes (k_fused_c<256, 8, 16> and
# k_tt_err's RK = 12 class on the paper's 256^4 ranks-10 shape), each after its plain run exited 0
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
python tools/rk16_one.py 5 > gpurun_out/rk16_one.log 2>&1; rc=$?; echo "rk16 rc $rc"; cat gpurun_out/rk16_one.log
if [ $rc -eq 0 ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused_c -c 1 -f \
    -o gpurun_out/fused_c_rk16_r2 python tools/rk16_one.py 5 > gpurun_out/ncu_full_rk16.log 2>&1; echo "ncu rk16 rc $?"
fi
python tools/err_pass256.py > gpurun_out/err_pass256.log 2>&1; rc=$?; echo "err256 rc $rc"; tail -3 gpurun_out/err_pass256.log
if [ $rc -eq 0 ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tt_err -c 1 -f \
    -o gpurun_out/tt_err_rk12_r2 python tools/err_pass256.py > gpurun_out/ncu_full_err256.log 2>&1; echo "ncu err256 rc $?"
fi
