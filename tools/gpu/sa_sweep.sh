for np in 0 2 4; do
  AT_SA_NP=$np timeout 300 python tools/sa_time.py cfg3 100 2>&1 | tail -1
done
AT_SA_NP=2 SA_CHAINS=8192 timeout 300 python tools/sa_time.py cfg3 100 2>&1 | tail -1
AT_SA_NP=2 timeout 300 python tools/sa_time.py cfg2 100 2>&1 | tail -1
