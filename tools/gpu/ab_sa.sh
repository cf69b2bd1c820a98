# A/B of the config-3 SA kernel: alternate library (AT_LIB=libautotvm_b200_alt.so) vs the current one
for lib in alt "" alt ""; do
L=paper_1805_08166_b200/libautotvm_b200${lib:+_$lib}.so
AT_LIB=$L timeout 600 python tools/sa_time.py cfg3 100 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib' or 'new', d['ms'], d['accept_digest'])"
done
timeout 600 python tools/sa_time.py cfg2 500 2>&1 | tail -1
