for i in 1 2; do timeout 600 python tools/bench_bcd.py config5 20 2>&1 | tail -1 | cut -c1-300; done
