"""Development probe for csrc/tc_f32.cu (TRG_TC_DEBUG dumps stage 0 of CTA 0)."""
import os
import sys
import numpy as np
sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import oracle_ref as orc
import paper_1901_01652_b200 as trg

np.set_printoptions(precision=4, linewidth=220, suppress=True)
os.environ["TRG_TC_DEBUG"] = "gpurun_out/tc_dbg.bin"
dims, K = (64, 40, 30), (16, 6, 5)
x = np.random.default_rng(0).standard_normal(dims).astype(np.float32)
proj, bases, ys = orc.sketch(x.astype(np.float64), K, 3)
got = trg.sketch(x, trg.ProjectionSpec(list(K), 3))
print("got[:4,:4]\n", got.sketches[0][:4, :4], "\nwant\n", ys[0][:4, :4])
d = np.fromfile("gpurun_out/tc_dbg.bin", dtype=np.float32)
print("A hi", d[:40])
print("A lo", d[256:296])
print("B hi", d[512:560])
print("B lo", d[640:688])
print("nt, tmem, kb, S", d[768:772])
X0 = x.reshape(64, -1, order="F")
print("X col 1152..: rows 0..7", X0[:8, 1152])
print("TMEM rows (q*32+lane) first 8 cols:")
for q in range(4):
    print(q, d[800 + q * 64: 800 + q * 64 + 16])
print("roundtrip", d[900:1028:8])
