import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from oracle import nm_oracle as O
from paper_2305_02678_b200 import neural
from paper_2305_02678_b200.latent import LatentPyramid
arch, mode, n = sys.argv[1], sys.argv[2], int(sys.argv[3])
rng = np.random.default_rng(0)
mat = neural.NeuralMaterial.create(neural.NeuralMaterialConfig(brdf_hidden=arch), rng)
mat.latent = LatentPyramid(O.random_pyramid(np.random.default_rng(0), 512, 512).levels)
qr = np.random.default_rng(1)
uv = qr.random((n, 2)).astype(np.float32); lod = (qr.random(n) * 9).astype(np.float32); urr = qr.random(n).astype(np.float32)
wi, wo = O.draw_direction_pairs(qr, n); wi, wo = wi.astype(np.float32), wo.astype(np.float32); u3 = qr.random((n, 3)).astype(np.float32)
t0 = time.time()
if mode == "eval": r = neural.eval_material(mat, uv, lod, wi, wo, urr, fp16=True)
elif mode == "sample": r = neural.sample_pdf(mat, uv, lod, urr, wi, u3)
else: r = neural.query(mat, uv, lod, urr, wi, wo, u3)
torch.cuda.synchronize()
print(arch, mode, n, "ok", time.time() - t0, flush=True)
