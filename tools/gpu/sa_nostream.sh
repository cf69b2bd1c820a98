for lib in paper_1805_08166_b200/libautotvm_b200.so paper_1805_08166_b200/libautotvm_b200_nostream.so; do
AT_LIB=$lib timeout 600 python tools/sa_time.py cfg3 100 2>&1 | tail -1
done
