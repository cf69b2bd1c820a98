# device bounds-checked variant (-DAT_CHECKS): the GPU parity suite and the all-kernels pass on it
export AT_LIB=$PWD/paper_1805_08166_b200/libautotvm_b200_checks.so
timeout 300 python tools/sanitize_run.py 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
