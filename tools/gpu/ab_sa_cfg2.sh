for lib in alt "" alt ""; do
L=paper_1805_08166_b200/libautotvm_b200${lib:+_$lib}.so
AT_LIB=$L timeout 600 python tools/sa_time.py cfg2 500 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-new}', 'cfg2', d['ms'], d['accept_digest'])"
AT_LIB=$L SA_CHAINS=8192 timeout 600 python tools/sa_time.py cfg3 100 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-new}', 'cfg3@8192', d['ms'], d['accept_digest'])"
done
