for eb in 0 1; do AT_SA_EB=$eb timeout 300 python tools/sa_time.py cfg3 100 2>&1 | tail -1; done
AT_SA_EB=1 SA_CHAINS=8192 timeout 300 python tools/sa_time.py cfg3 100 2>&1 | tail -1
