"""Build the -DAT_CHECKS variant (device bounds checks, see at_common.cuh AT_DCHECK) as
paper_1805_08166_b200/libautotvm_b200_checks.so; run anything against it with AT_LIB=<that path>."""
import sys
sys.path.insert(0, ".")
from paper_1805_08166_b200 import build
print(build.build(defines=("-DAT_CHECKS",), lib=build.PKG / "libautotvm_b200_checks.so"))
