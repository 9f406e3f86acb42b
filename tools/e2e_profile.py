"""cProfile of the drop-in eval_material call on the C2 batch (host overhead)."""
import cProfile, os, pstats, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2305_02678_b200 import neural, synth
dev = torch.device("cuda", 0)
mat = synth.material("2x32", 4096, 4096, seed=0, device=dev)
n = 1920 * 1080
q = synth.queries(n, mat.latent.n_levels, seed=1, device=dev)
hq = {k: v.cpu().numpy() for k, v in q.items()}
for _ in range(3):
    neural.eval_material(mat, hq["uv"], hq["lod"], hq["wi"], hq["wo"], hq["u_rr"], fp16=True)
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    neural.eval_material(mat, hq["uv"], hq["lod"], hq["wi"], hq["wo"], hq["u_rr"], fp16=True)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
