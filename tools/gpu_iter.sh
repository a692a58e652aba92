timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/c2_launches.csv python tools/prof_config2.py > /dev/null 2>&1; echo "ncu rc $?"
