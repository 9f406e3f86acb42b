"""Training kernels only, for compute-sanitizer: forward/backward of a
32-wide and a 64-wide network at an odd and an aligned batch (the
register-fed and the TMA-fed tensor-core dW/db, the float64 and float
SMEM weight copies), and the texel-gradient scatter with random levels (the
SMEM-summed coarse tail included); partial tiles included."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from oracle import nm_oracle as O
from paper_2305_02678_b200 import mlp, neural, train
from paper_2305_02678_b200.latent import LatentPyramid

rng = np.random.default_rng(0)
n = 1000 + 37
for rows in (n, 4096):  # odd batch: register-fed dW/db; aligned batch: the TMA-fed one
    for dims in ((20, 32, 32, 3), (20, 64, 64, 64, 3), (11, 32, 32, 32, 9), (64,) + (64,) * 8 + (3,)):
        net = mlp.Mlp.create(dims, rng)
        out, cache = train.forward_cached(net, rng.normal(size=(rows, dims[0])).astype(np.float32))
        train.backward(net, cache, rng.normal(size=(rows, dims[-1])).astype(np.float32))
mat = neural.NeuralMaterial.create(neural.NeuralMaterialConfig(), rng)
mat.latent = LatentPyramid(O.random_pyramid(rng, 64, 32).levels)
uv = rng.random((n, 2)).astype(np.float32)
lv = rng.integers(0, mat.latent.n_levels, n)
mat.latent.accumulate_texel_grads(mat.latent.zero_grads(), uv, lv, rng.normal(size=(n, 8)).astype(np.float32))
print("sanitize_train ok")
