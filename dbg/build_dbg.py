"""Build dbg/libautotvm_b200.so with extra -D flags (instrumented kernels), e.g.
    python dbg/build_dbg.py -DAT_FIT_TIMING"""
import subprocess, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1805_08166_b200 import build as b
out = Path(__file__).resolve().parent
objs = []
for src in b.SOURCES:
    o = out / (Path(src).stem + ".o")
    subprocess.check_call([b.NVCC, *b.FLAGS, *sys.argv[1:], "-c", str(b.CSRC / src), "-o", str(o)])
    objs.append(str(o))
subprocess.check_call([b.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(out / "libautotvm_b200.so"),
                       *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"])
print(out / "libautotvm_b200.so")
