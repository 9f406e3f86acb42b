"""Calibrate the fast kernel's T.w error bound.

The pipelined eval kernel computes the decoder's direction inputs T.wi, T.wo
in fp32 from the tensor-core frame layer; a value within tw_delta x kappa
(kappa = the frame's conditioning, 1 + |rt|_1/|n x rt|) of an fp16 rounding
midpoint is resolved exactly.  This tool dumps the fast fp32 values
(nm_eval_debug_tw) for C2-sized batches, recomputes them in the reference's
arithmetic with the oracle (fp32 BLAS frame layer, float64 frames and
transforms, narrowed to fp32), and reports max |fast - exact| / kappa, the
share of rows queued at the built-in bound, and rows whose fp16 inputs
differ without being queued (must be 0).

    python tools/tw_calibrate.py [--n 2073600] [--seeds 4]
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import nm_oracle as O  # noqa: E402
from paper_2305_02678_b200 import _lib, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1920 * 1080)
    ap.add_argument("--seeds", type=int, default=4)
    ap.add_argument("--delta", type=float, default=2.5e-7)
    args = ap.parse_args()
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    worst, flagged, total, missed, diff_rows = 0.0, 0, 0, 0, 0
    q_all = []
    for seed in range(args.seeds):
        mat = synth.material("2x32", 4096, 4096, seed=seed, device=dev)
        h = mat.device_material(dev)
        q = synth.queries(args.n, mat.latent.n_levels, seed=100 + seed, device=dev)
        n = args.n
        rgb = torch.empty((n, 3), device=dev)
        dbg = torch.empty((n, 14), device=dev)
        z = torch.empty((n, 8), device=dev)
        st = torch.cuda.current_stream().cuda_stream
        _lib.check(lib.nm_eval_debug_tw(h.ptr, n, q["uv"].data_ptr(), q["lod"].data_ptr(), 1,
                                        q["u_rr"].data_ptr(), q["wi"].data_ptr(), q["wo"].data_ptr(),
                                        rgb.data_ptr(), dbg.data_ptr(), st))
        _lib.check(lib.nm_fetch(h.ptr, n, q["uv"].data_ptr(), q["lod"].data_ptr(), 1, q["u_rr"].data_ptr(),
                                z.data_ptr(), None, None, None, st))
        torch.cuda.synchronize()
        d = dbg.cpu().numpy()
        zh = z.cpu().numpy()
        wi = q["wi"].cpu().numpy().astype(np.float64)
        wo = q["wo"].cpu().numpy().astype(np.float64)
        frame = O.quantize(O.Net([(l.w, l.b, l.act) for l in mat.frame_layer.layers]))
        raw = frame.forward(zh)
        fr = O.frames_from_raw(raw)
        ex = np.concatenate([O.frame_transform(fr, wi), O.frame_transform(fr, wo)], 1).astype(np.float32)
        fast = d[:, :12]
        kap = np.concatenate([np.repeat(d[:, 12:13], 3, 1), np.repeat(d[:, 13:14], 3, 1)], 1)
        kap = np.concatenate([kap, kap], 1)  # [ti f1, ti f2, to f1, to f2]
        err = np.abs(fast.astype(np.float64) - ex) / kap
        finite = np.isfinite(kap)
        worst = max(worst, float(err[finite].max()))
        dl = np.float32(args.delta) * kap.astype(np.float32)
        near = ((fast + dl).astype(np.float16) != (fast - dl).astype(np.float16)) | ~finite
        qflag = near.any(1)
        differ = (fast.astype(np.float16) != ex.astype(np.float16))
        flagged += int(qflag.sum())
        total += n
        diff_rows += int(differ.any(1).sum())
        missed += int((differ.any(1) & ~qflag).sum())
        q_all.append(np.quantile(err[finite], [0.5, 0.99, 0.9999]).tolist())
        print(json.dumps({"seed": seed, "max_err_over_kappa": float(err[finite].max()),
                          "q50_q99_q9999": q_all[-1], "rows_queued": float(qflag.mean()),
                          "rows_fp16_differ": float(differ.any(1).mean()),
                          "missed": int((differ.any(1) & ~qflag).sum())}), flush=True)
    print(json.dumps({"rows": total, "max_err_over_kappa": worst, "delta": args.delta,
                      "margin": args.delta / worst, "queued_share": flagged / total,
                      "fp16_differ_share": diff_rows / total, "missed": missed}))


if __name__ == "__main__":
    main()
