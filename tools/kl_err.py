import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from conftest import load_golden
from test_gpu_kl import _mat, TAGS
from paper_2305_02678_b200 import train
g = load_golden("kl")
for tag in TAGS:
    mat = _mat(g, tag)
    loss, grads = train.sampler_loss_and_grads(mat, g[f"{tag}_z"], g[f"{tag}_wi"], None, us=(g[f"{tag}_ud"], g[f"{tag}_us"]))
    want = float(g[f"{tag}_loss"])
    errs = []
    for i, (dw, db) in enumerate(grads):
        for a, w in ((dw, g[f"{tag}_dw{i}"]), (db, g[f"{tag}_db{i}"])):
            errs.append(np.abs(a - w).max() / np.abs(w).max())
    print(tag, "loss", loss, want, "rel %.2e" % (abs(loss - want) / abs(want)), "grad max rel-to-max %.2e" % max(errs))
