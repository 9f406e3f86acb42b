import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from conftest import load_golden
from test_gpu_parity import _train_net
g = load_golden("train")
for tag in ["brdf", "samp", "wide", "deep"]:
    net = _train_net(g, tag)
    out, cache = net.forward_cached(g[f"{tag}_x"])
    grads, dx = net.backward(cache, g[f"{tag}_g"])
    e = max(max(np.abs(dw - g[f"{tag}_dw{i}"]).max() / np.abs(g[f"{tag}_dw{i}"]).max(),
                np.abs(db - g[f"{tag}_db{i}"]).max() / np.abs(g[f"{tag}_db{i}"]).max()) for i, (dw, db) in enumerate(grads))
    print(tag, "dW/db max err rel-to-max %.2e" % e)
