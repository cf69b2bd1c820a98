for lib in alt spec1 spec3 "" spec5 spec7; do
L=paper_1805_08166_b200/libautotvm_b200${lib:+_$lib}.so
echo "== $L"; AT_LIB=$L timeout 600 python tools/sa_time.py cfg3 100 2>&1 | tail -1
done
AT_LIB=paper_1805_08166_b200/libautotvm_b200_alt.so timeout 600 python tools/sa_time.py cfg2 500 2>&1 | tail -1
timeout 600 python tools/sa_time.py cfg2 500 2>&1 | tail -1
