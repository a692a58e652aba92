timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_skinny_tc16 -c 2 -o gpurun_out/tc16_packed python tools/prof_config5.py > gpurun_out/ncu_tc16b.log 2>&1; echo rc $?
