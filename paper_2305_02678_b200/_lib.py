"""ctypes binding of libnmq.so (include/nmq.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_2305_02678_b200.build``).  There is no CPU fallback: if the
library is missing, importing the query API raises immediately.
"""

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NMQ_LIB") or os.path.join(_HERE, "libnmq.so")

NM_OK = 0
NM_ERR_INVALID = -1
NM_ERR_CUDA = -2
NM_ERR_UNSUPPORTED = -3

NM_QUERY_EVAL, NM_QUERY_SAMPLE_PDF, NM_QUERY_FULL = 0, 1, 2
NM_MULTI_DIVERGENT = 0
NM_MULTI_BINNED = 1
NM_MULTI_BINNED_ASYNC = 2
NM_KL_SCRATCH = 17  # doubles per row of the KL-loss scratch (include/nmq.h)

c_float_p = ctypes.c_void_p  # device pointers are passed as raw addresses
c_i64 = ctypes.c_int64
c_i32 = ctypes.c_int32


class NetDesc(ctypes.Structure):
    _fields_ = [
        ("n_layers", ctypes.c_int32),
        ("fan_in", ctypes.POINTER(ctypes.c_int32)),
        ("fan_out", ctypes.POINTER(ctypes.c_int32)),
        ("act", ctypes.POINTER(ctypes.c_int32)),
        ("packed", ctypes.POINTER(ctypes.c_uint16)),
        ("weights", ctypes.POINTER(ctypes.c_float)),
    ]


class MaterialDesc(ctypes.Structure):
    _fields_ = [
        ("channels", ctypes.c_int32),
        ("use_frames", ctypes.c_int32),
        ("n_frames", ctypes.c_int32),
        ("albedo_head", ctypes.c_int32),
        ("sampler_isotropic", ctypes.c_int32),
        ("frame", NetDesc),
        ("brdf", NetDesc),
        ("sampler", NetDesc),
        ("width", ctypes.c_int32),
        ("height", ctypes.c_int32),
        ("n_levels", ctypes.c_int32),
        ("latent", ctypes.c_void_p),
        ("latent_fp32", ctypes.c_int32),
        ("latent_on_device", ctypes.c_int32),
        ("precise", ctypes.c_int32),
    ]


class MaterialInfo(ctypes.Structure):
    _fields_ = [
        ("device", ctypes.c_int32),
        ("n_levels", ctypes.c_int32),
        ("latent_texels", ctypes.c_int64),
        ("latent_bytes", ctypes.c_int64),
        ("weight_bytes", ctypes.c_int32),
        ("brdf_width", ctypes.c_int32),
        ("sampler_width", ctypes.c_int32),
    ]


# name -> (restype, argtypes); must match include/nmq.h exactly
SIGNATURES = {
    "nm_material_create": (c_i32, [ctypes.POINTER(MaterialDesc), c_i32, ctypes.POINTER(ctypes.c_void_p)]),
    "nm_material_destroy": (c_i32, [ctypes.c_void_p]),
    "nm_material_info_get": (c_i32, [ctypes.c_void_p, ctypes.POINTER(MaterialInfo)]),
    "nm_material_levels": (c_i32, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "nm_material_latent_ptr": (ctypes.c_void_p, [ctypes.c_void_p]),
    "nm_fetch": (c_i32, [ctypes.c_void_p, c_i64, c_float_p, c_float_p, c_i32, c_float_p,
                         c_float_p, ctypes.c_void_p, ctypes.c_void_p, c_float_p, ctypes.c_void_p]),
    "nm_eval": (c_i32, [ctypes.c_void_p, c_i64, c_float_p, c_float_p, c_i32, c_float_p, c_float_p,
                        c_float_p, c_float_p, c_float_p, ctypes.c_void_p, ctypes.c_void_p]),
    "nm_eval_z": (c_i32, [ctypes.c_void_p, c_i64, c_float_p, c_float_p, c_float_p, c_float_p,
                          c_float_p, ctypes.c_void_p]),
    "nm_infer_proxy": (c_i32, [ctypes.c_void_p, c_i64, c_float_p, c_float_p, c_float_p,
                               ctypes.c_void_p]),
    "nm_sample": (c_i32, [c_i64, c_float_p, c_float_p, c_float_p, c_float_p, ctypes.c_void_p]),
    "nm_pdf": (c_i32, [c_i64, c_float_p, c_float_p, c_float_p, c_float_p, ctypes.c_void_p]),
    "nm_sample_pdf": (c_i32, [ctypes.c_void_p, c_i64, c_float_p, c_float_p, c_i32, c_float_p,
                              c_float_p, c_float_p, c_float_p, c_float_p, c_float_p,
                              ctypes.c_void_p, ctypes.c_void_p]),
    "nm_query": (c_i32, [ctypes.c_void_p, c_i64, c_float_p, c_float_p, c_i32, c_float_p,
                         c_float_p, c_float_p, c_float_p, c_float_p, c_float_p, c_float_p,
                         ctypes.c_void_p, ctypes.c_void_p]),
    "nm_multi_workspace_bytes": (ctypes.c_size_t, [c_i64, c_i32]),
    "nm_eval_multi": (c_i32, [ctypes.c_void_p, c_i32, c_i64, ctypes.c_void_p, c_float_p, c_float_p,
                              c_i32, c_float_p, c_float_p, c_float_p, c_float_p, c_i32,
                              ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "nm_sample_pdf_multi": (c_i32, [ctypes.c_void_p, c_i32, c_i64, ctypes.c_void_p, c_float_p, c_float_p, c_i32,
                                    c_float_p, c_float_p, c_float_p, c_float_p, c_float_p, c_float_p, c_i32,
                                    ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "nm_query_multi": (c_i32, [ctypes.c_void_p, c_i32, c_i64, ctypes.c_void_p, c_float_p, c_float_p, c_i32,
                               c_float_p, c_float_p, c_float_p, c_float_p, c_float_p, c_float_p, c_float_p, c_i32,
                               ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "nm_fetch_f64": (c_i32, [ctypes.c_void_p, c_i64, ctypes.c_void_p, ctypes.c_void_p, c_i32, ctypes.c_void_p,
                             ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "nm_query_f64": (c_i32, [ctypes.c_void_p, c_i32, c_i64] + [ctypes.c_void_p] * 14),
    "nm_eval_z_f64": (c_i32, [ctypes.c_void_p, c_i64] + [ctypes.c_void_p] * 6),
    "nm_eval_host_ref": (c_i32, [ctypes.c_void_p, c_i64, ctypes.c_void_p, ctypes.c_void_p, c_i32]
                         + [ctypes.c_void_p] * 6 + [c_i64, ctypes.c_void_p]),
    "nm_decoder_inputs": (c_i32, [ctypes.c_void_p, c_i64] + [ctypes.c_void_p] * 7),
    "nm_eval_spp": (c_i32, [ctypes.c_void_p, c_i64, c_float_p, c_float_p, c_i32, c_float_p, c_float_p,
                            c_float_p, c_i32, c_float_p, ctypes.c_void_p]),
    "nm_fetch_trilinear": (c_i32, [ctypes.c_void_p, c_i64, c_float_p, c_float_p, c_i32, c_float_p,
                                   ctypes.c_void_p, ctypes.c_void_p]),
    "nm_eval_host": (c_i32, [ctypes.c_void_p, c_i64, c_float_p, c_float_p, c_i32, c_float_p,
                             c_float_p, c_float_p, c_float_p, c_float_p, ctypes.c_void_p, c_i64,
                             ctypes.c_void_p]),
    "nm_texel_grads": (c_i32, [ctypes.c_void_p, c_i64, c_float_p, ctypes.c_void_p, c_float_p, c_float_p,
                               ctypes.c_void_p]),
    "nm_mlp_create": (c_i32, [ctypes.c_void_p, c_i32, ctypes.c_void_p]),
    "nm_mlp_set_weights": (c_i32, [ctypes.c_void_p, ctypes.c_void_p]),
    "nm_mlp_destroy": (c_i32, [ctypes.c_void_p]),
    "nm_mlp_params": (c_i32, [ctypes.c_void_p]),
    "nm_mlp_cache_bytes": (ctypes.c_size_t, [ctypes.c_void_p, c_i64]),
    "nm_mlp_forward_cached": (c_i32, [ctypes.c_void_p, c_i64, c_float_p, c_float_p, ctypes.c_void_p,
                                      ctypes.c_void_p]),
    "nm_mlp_backward": (c_i32, [ctypes.c_void_p, c_i64, ctypes.c_void_p, c_float_p, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_void_p]),
    "nm_kl_sample": (c_i32, [c_i64, c_i32, c_i32, c_i32] + [ctypes.c_void_p] * 9),
    "nm_kl_target": (c_i32, [c_i64, c_i32] + [ctypes.c_void_p] * 6),
    "nm_kl_target_dir": (c_i32, [c_i64, c_i32, c_i32] + [ctypes.c_void_p] * 6),
    "nm_kl_grad": (c_i32, [c_i64, c_i32] + [ctypes.c_void_p] * 8),
    "nm_footprint_level": (c_i32, [c_i64, ctypes.c_void_p, c_i32, ctypes.c_void_p, ctypes.c_void_p]),
    "nm_cone_level": (c_i32, [c_i64, c_float_p, c_float_p, c_float_p, c_float_p, c_float_p, c_i32,
                              c_i32, c_float_p, ctypes.c_void_p]),
    "nm_last_error": (ctypes.c_char_p, []),
    "nm_version": (c_i32, []),
    "nm_launch_count": (c_i64, []),
    "nm_set_kernel_path": (c_i32, [c_i32]),
    "nm_last_kernel_path": (c_i32, []),
    "nm_set_tw_margin": (c_i32, [ctypes.c_float]),
    "nm_eval_debug_tw": (c_i32, [ctypes.c_void_p, c_i64, c_float_p, c_float_p, c_i32, c_float_p, c_float_p,
                                 c_float_p, c_float_p, c_float_p, ctypes.c_void_p]),
}

_lib = None


class NmqError(RuntimeError):
    pass


def load():
    """Load libnmq.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the query path has no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        if os.environ.get("NMQ_LIB") and not hasattr(lib, name):
            continue  # an experimental / older build (NMQ_LIB) may lack newer entry points
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if os.environ.get("NMQ_KERNEL_PATH"):  # experiments: force a kernel family (see nmq.h)
        lib.nm_set_kernel_path(int(os.environ["NMQ_KERNEL_PATH"]))
    if os.environ.get("NMQ_TW_MARGIN"):  # experiments: exact-rounding queue bound (see nmq.h)
        lib.nm_set_tw_margin(float(os.environ["NMQ_TW_MARGIN"]))
    _lib = lib
    return lib


def check(rc, what=""):
    """Map a status code to the reference's exception types (ValueError for
    shape/argument problems, mlp.py:85)."""
    if rc == NM_OK:
        return
    msg = load().nm_last_error().decode("utf-8", "replace")
    if rc == NM_ERR_INVALID:
        raise ValueError(msg)
    if rc == NM_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise NmqError(f"{what}: {msg}" if what else msg)
