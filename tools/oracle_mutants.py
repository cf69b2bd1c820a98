"""Mutation check of the oracle's pins: plant plausible mistakes (a dropped term, a wrong sign, index or
operand, a flipped comparison) in a copy of oracle/oracle.c and confirm that `tests/test_oracle_pins.py`
(-m "not gpu") turns red for each.  Nothing in the repo is modified: every mutant runs in a scratch copy
of the tracked files.

    python tools/oracle_mutants.py [-k substring]   -> one line per mutant, summary at the end
"""
import os
import shutil
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

# (name, paper passage the line implements, original text, mutated text)
MUTANTS = [
    ("metropolis: sign of -d/T", "Alg. 1 P:152-153", "float a = -(d / temps[st]);", "float a = (d / temps[st]);"),
    ("metropolis: Philox word 3 for u", "Q20 / P:187", "float u = (float)(r[2] >> 8)", "float u = (float)(r[3] >> 8)"),
    ("metropolis: T ignored", "Alg. 1 P:152-153", "float a = -(d / temps[st]);", "float a = -d;"),
    ("gbt: x <= theta goes left", "Q18 / P:129-133", "node = (x[f] < th) ? 2 * node + 1 : 2 * node + 2;",
     "node = (x[f] <= th) ? 2 * node + 1 : 2 * node + 2;"),
    ("gbt: children swapped", "Q18", "node = (x[f] < th) ? 2 * node + 1 : 2 * node + 2;",
     "node = (x[f] < th) ? 2 * node + 2 : 2 * node + 1;"),
    ("refit gain: lambda dropped in the parent term", "Eq. 2 / Q37",
     "- G * G / (H + lam);", "- G * G / H;"),
    ("refit gain: right child dropped", "Q37", "(GL * GL / (HL + lam) + GR * GR / (HR + lam)) - G * G / (H + lam);",
     "(GL * GL / (HL + lam)) - G * G / (H + lam);"),
    ("refit: gradient sign", "Eq. 2 P:176-179", "g[i] -= 2 * q;", "g[i] += 2 * q;"),
    ("refit: sigmoid argument transposed", "Eq. 2 P:178", "float d = pred[j] - pred[i];", "float d = pred[i] - pred[j];"),
    ("refit: leaf sign", "Q37", "tl[l] = (float)(-(eta * (G / (H + lam))));", "tl[l] = (float)(eta * (G / (H + lam)));"),
    ("refit: curvature term", "Eq. 2", "float hh = rho * (1.0f - rho);", "float hh = rho;"),
    ("select: coverage counts covered knobs", "Eq. 3 P:196-201", "if (!covered) ++newcov;", "if (covered) ++newcov;"),
    ("select: sign of z", "Eq. 3", "double gain = (-z) + (double)alpha * (double)newcov;",
     "double gain = z + (double)alpha * (double)newcov;"),
    ("select: alpha dropped", "Eq. 3", "double gain = (-z) + (double)alpha * (double)newcov;", "double gain = (-z);"),
    ("features: relation threshold <= beta", "P:256 / Q10", "if (rows[k].touch[b] < ((uint64_t)1 << t)) {",
     "if (rows[k].touch[b] <= ((uint64_t)1 << t)) {"),
    ("features: stride slot gets the touch count", "Appendix A / P:646", "z[12 + 3 * b] = (float)rows[k].stride[b];",
     "z[12 + 3 * b] = (float)rows[k].touch[b];"),
    ("features: loop product misses the last loop", "Appendix A", "for (int k = 0; k < ns->n; ++k) total *= ns->ext[k];",
     "for (int k = 0; k + 1 < ns->n; ++k) total *= ns->ext[k];"),
    ("exp_det: one Taylor term dropped", "Q22", "p = fmaf(p, r, f_from_bits(0x3C088889u)); /* 1/120 */",
     "/* 1/120 dropped */"),
    ("exp_det: ln2 low part dropped", "Q22", "r = fmaf(-n, ln2_lo, r);", "/* lo dropped */"),
    ("top-k: ties by descending index", "O10 / Q24", "if (x->idx < y->idx) return -1;\n    if (x->idx > y->idx) return 1;",
     "if (x->idx > y->idx) return -1;\n    if (x->idx < y->idx) return 1;"),
    ("top-k: descending energy", "O10", "if (x->E < y->E) return -1;\n    if (x->E > y->E) return 1;",
     "if (x->E > y->E) return -1;\n    if (x->E < y->E) return 1;"),
    ("select: eps count floor", "Q26", "int32_t n_rand = (int32_t)ceilf(eb);", "int32_t n_rand = (int32_t)floorf(eb);"),
    ("space: knob 0 slowest", "S:138-146", "choices[j] = (int)(idx % (uint64_t)sp->radix[j]);\n        idx /= (uint64_t)sp->radix[j];",
     "choices[sp->n_knobs - 1 - j] = (int)(idx % (uint64_t)sp->radix[sp->n_knobs - 1 - j]);\n        idx /= (uint64_t)sp->radix[sp->n_knobs - 1 - j];"),
    ("features: reuse inverted", "P:636 / Q6", "r->reuse[b] = (float)r->bottom_up / (float)r->touch[b];",
     "r->reuse[b] = (float)r->touch[b] / (float)r->bottom_up;"),
    ("features: top-down includes the loop itself", "Q9", "for (int l = 0; l < k; ++l) r->top_down *= ns->ext[l];",
     "for (int l = 0; l <= k; ++l) r->top_down *= ns->ext[l];"),
    ("refit: min_child_weight ignored", "Q37", "if (HL < mcw || HR < mcw) continue;", "if (HL < 0 || HR < 0) continue;"),
    ("refit: split tie takes the later split", "Q37", "if (bf[q] < 0 || gain > bg[q])", "if (bf[q] < 0 || gain >= bg[q])"),
]


def tracked_copy(dst: Path) -> None:
    files = subprocess.run(["git", "ls-files"], cwd=ROOT, capture_output=True, text=True, check=True).stdout.split()
    for f in files:
        src = ROOT / f
        if not src.is_file():
            continue
        out = dst / f
        out.parent.mkdir(parents=True, exist_ok=True)
        shutil.copy2(src, out)


def main() -> int:
    sel = sys.argv[sys.argv.index("-k") + 1] if "-k" in sys.argv else ""
    caught = missed = 0
    with tempfile.TemporaryDirectory() as td:
        base = Path(td) / "repo"
        tracked_copy(base)
        src = (base / "oracle" / "oracle.c").read_text()
        for name, passage, old, new in MUTANTS:
            if sel and sel not in name:
                continue
            n = src.count(old)
            if n != 1:
                print(f"SKIP    {name}: pattern found {n} times")
                continue
            (base / "oracle" / "oracle.c").write_text(src.replace(old, new))
            for so in (base / "oracle").glob("liboracle.so*"):
                so.unlink()
            t0 = time.time()
            r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_pins.py", "-x", "-q", "-m", "not gpu",
                                "-p", "no:cacheprovider"], cwd=base, capture_output=True, text=True,
                               env={**os.environ, "PYTHONPATH": str(base)})
            failed = [l for l in r.stdout.splitlines() if l.startswith("FAILED")]
            ok = r.returncode != 0
            caught += ok
            missed += not ok
            print(f"{'CAUGHT' if ok else 'MISSED'}  {name} ({passage}) {time.time() - t0:.0f}s"
                  + (f" <- {failed[0][7:].split(' - ')[0]}" if failed else ""), flush=True)
        (base / "oracle" / "oracle.c").write_text(src)
    print(f"{caught} caught, {missed} missed")
    return 0 if missed == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
