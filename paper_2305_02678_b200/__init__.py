"""B200-native (sm_100a) neural-material query path — a drop-in for the
query hot path of the reference ``neuralmat`` package (arXiv 2305.02678).

Modules mirror the reference's names: ``latent`` (LatentPyramid.fetch),
``neural`` (eval_brdf / eval_material / infer_proxy / archives),
``proxy`` (ProxyParams / sample / pdf), ``mlp`` (weights + fp16 packing),
``render`` (LoD from ray cones), ``train`` (training-side kernels:
forward_cached / backward, texel-gradient scatter).
All queries run in the CUDA kernels of ``libnmq.so`` (include/nmq.h).
"""

from . import mlp, latent, proxy, neural, render, train  # noqa: F401
from .latent import LatentPyramid  # noqa: F401
from .neural import (NeuralMaterial, NeuralMaterialConfig, eval_brdf, eval_material,  # noqa: F401
                     eval_material_multi,
                     infer_proxy, load_archive, query, sample_pdf, save_archive)

__version__ = "0.1.0"
