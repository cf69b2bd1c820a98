"""Per-block level work of the fused forest on config 3's |D| = 1536 (instrumented build with
-DAT_FIT_TIMING -DAT_FIT_BLOCKS_DUMP=1): which blocks are slow -- those sharing an SM with two others, or
those whose feature has many cuts?  Prints a summary of work ns/tree by blocks-per-SM and by cut count."""
import collections, os, subprocess, sys
sys.path.insert(0, ".")
if os.environ.get("FTB_CHILD") != "1":
    from paper_1805_08166_b200 import build
    build.build(defines=("-DAT_FIT_TIMING", "-DAT_FIT_BLOCKS_DUMP=1"), lib=build.PKG / "libautotvm_b200_fitblk.so")
    out = subprocess.run([sys.executable, __file__], env={**os.environ, "FTB_CHILD": "1"}, capture_output=True,
                         text=True).stdout
    rows = [l.split()[1:] for l in out.splitlines() if l.startswith("FTBLK")]
    rows = [(int(b), int(sm), int(f), int(nc), int(w), int(gn)) for b, sm, f, nc, w, gn in rows]
    per_sm = collections.Counter(r[1] for r in rows)
    by_k = collections.defaultdict(list)
    for r in rows:
        by_k[per_sm[r[1]]].append(r[4])
    for k, v in sorted(by_k.items()):
        print(f"blocks on SMs hosting {k}: n={len(v)} work ns/tree mean {sum(v) / len(v):.0f} max {max(v)}")
    rows.sort(key=lambda r: r[3])
    q = len(rows) // 4
    for i in range(4):
        part = rows[i * q:(i + 1) * q] if i < 3 else rows[3 * q:]
        print(f"cut-count quartile {i}: ncuts {part[0][3]}..{part[-1][3]} work mean {sum(r[4] for r in part) / len(part):.0f}"
              f" gains mean {sum(r[5] for r in part) / len(part):.0f}")
    print("block -> sm (first 8):", [(r[0], r[1]) for r in sorted(rows)[:8]])
    sys.exit(0)
import numpy as np, torch
from paper_1805_08166_b200 import at, build, synth
at.LIB_PATH = build.PKG / "libautotvm_b200_fitblk.so"
wls, nper = synth.ALL_RESNET, 128
sp = at.Space(wls)
n = 12 * nper
key = (np.arange(n) % 12).astype(np.uint16)
sizes = np.array([sp.size(w) for w in range(12)], dtype=np.uint64)
loc = synth.uniform_indices(1 << 62, n, seed=1806) % sizes[key]
idx = loc + np.array(sp.offsets[:12], dtype=np.uint64)[key]
X = sp.features(torch.from_numpy(idx.view(np.int64)).cuda())
c = torch.from_numpy(synth.labels(X[:, :n].T.cpu().numpy(), seed=1807)).cuda()
k = torch.from_numpy(key.view(np.int16)).cuda()
at.gbt_fit_hist(X, n, c, k, n_trees=100, depth=6)
torch.cuda.synchronize()
