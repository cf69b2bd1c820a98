for lib in "" spec0 spec2 "" spec0 spec2; do
L=paper_1805_08166_b200/libautotvm_b200${lib:+_$lib}.so
AT_LIB=$L timeout 600 python tools/sa_time.py cfg3 100 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-spec1}', d['ms'], d['accept_digest'])"
done
