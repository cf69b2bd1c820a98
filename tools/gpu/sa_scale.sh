for G in 1 2; do AT_SA_GRP=$G timeout 300 python tools/sa_time.py cfg2 100 2>&1 | tail -1; done
for C in 4096 2048; do for G in 1 2; do
  SA_CHAINS=$C AT_SA_GRP=$G timeout 300 python tools/sa_time.py cfg3 100 2>&1 | tail -1
done; done
