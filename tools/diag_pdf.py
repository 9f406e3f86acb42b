"""Diagnostic: where does the decoupled pdf error come from?"""
import sys
import numpy as np
sys.path.insert(0, "tests")
sys.path.insert(0, ".")
from conftest import load_golden, rel_err  # noqa
from test_gpu_parity import our_material  # noqa
from oracle import nm_oracle as O  # noqa
from paper_2305_02678_b200 import neural, proxy  # noqa

g = load_golden(sys.argv[1] if len(sys.argv) > 1 else "c1_2x32")
mat = our_material(g)
p = neural.infer_proxy(mat, g["z"].astype(np.float32), g["wi"], fp16=True)
ours = p.as_array()
ref = g["params"]
names = ["wd", "ws", "mdx", "mdy", "ax", "ay", "rho", "msx", "msy"]
for k, nm in enumerate(names):
    r = np.abs(ours[:, k] - ref[:, k]) / (np.abs(ref[:, k]) + 1e-30)
    print(f"{nm}: max relerr {r.max():.3e} mean {r.mean():.3e}  absmax {np.abs(ours[:, k]-ref[:, k]).max():.3e}")
pw = proxy.pdf(p, g["wi"], g["ws"])
r = rel_err(pw, g["pdf_ws"])
i = int(np.argmax(r))
print("worst", i, "ours", pw[i], "ref", g["pdf_ws"][i])
print("params ours", ours[i])
print("params ref ", ref[i])
# oracle pdf with our params (f64) vs ref params
P = lambda b: O.Proxy(b[:, 0], b[:, 1], b[:, 2:4], b[:, 4:6], b[:, 6], b[:, 7:9])
wi = g["wi"][i:i + 1].astype(np.float64)
ws = g["ws"][i:i + 1]
print("oracle f64 pdf with our params:", O.pdf(P(ours[i:i + 1]), wi, ws), " with ref params:", O.pdf(P(ref[i:i + 1]), wi, ws))
print("kernel pdf with ref params (fp32):", proxy.pdf(proxy.ProxyParams(*[ref[i:i+1, s] for s in (0, 1, slice(2, 4), slice(4, 6), 6, slice(7, 9))]), wi, ws))
