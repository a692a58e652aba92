for v in 0 1 0 1; do echo "== 1cta $v"; NTT_C_1CTA=$v timeout 300 python tools/persist_trace.py 2>&1 | sed -n 2,3p; done
