"""Network parameter containers and the fp16 quantization the GPU consumes.

Host-side only: these classes hold weights; nothing here evaluates a
network (the query path runs on the GPU, see ``neural.py``).  Names and
semantics mirror the reference's ``neuralmat.mlp``:

* ``Mlp.create`` — He-style fan-in uniform init consuming the RNG layer by
  layer exactly like ``mlp.py:57-69`` (so a seeded synthetic material is the
  same material the reference would build);
* ``quantize`` — clamp to +-65504 (counted), RNE to fp16, packed per output
  neuron as ``[w_row, bias]`` in layer order (``mlp.py:214-233``); this
  packed buffer is exactly what ``nm_material_create`` takes;
* ``write_blob`` / ``read_blob`` — the ``NMWB0001`` weight blob
  (``mlp.py:241-273``), byte-compatible with the reference.
"""

import io
import struct

import numpy as np

LEAKY_SLOPE = 0.01
FP16_MAX = 65504.0
ACT_LINEAR = "linear"
ACT_LEAKY = "leaky_relu"
ACT_CODES = {ACT_LINEAR: 0, ACT_LEAKY: 1}
ACT_NAMES = {0: ACT_LINEAR, 1: ACT_LEAKY}
BLOB_MAGIC = b"NMWB0001"


class Layer:
    __slots__ = ("w", "b", "act")

    def __init__(self, w, b, act):
        if act not in ACT_CODES:
            raise ValueError(f"unknown activation {act!r}")
        self.w = np.ascontiguousarray(w, dtype=np.float32)
        self.b = np.ascontiguousarray(b, dtype=np.float32)
        self.act = act


class Mlp:
    """fp32 master parameters of one network (rows = output neurons)."""

    def __init__(self, layers):
        for prev, nxt in zip(layers, layers[1:]):
            if nxt.w.shape[1] != prev.w.shape[0]:
                raise ValueError("layer dimensions do not chain")
        self.layers = list(layers)

    @classmethod
    def create(cls, sizes, rng, hidden_act=ACT_LEAKY, out_act=ACT_LINEAR, weight_scale=1.0):
        layers = []
        n = len(sizes) - 1
        for i in range(n):
            fan_in, fan_out = sizes[i], sizes[i + 1]
            lim = weight_scale * np.sqrt(6.0 / fan_in)
            w = rng.uniform(-lim, lim, size=(fan_out, fan_in))
            layers.append(Layer(w, np.zeros(fan_out), out_act if i == n - 1 else hidden_act))
        return cls(layers)

    @property
    def in_dim(self):
        return self.layers[0].w.shape[1]

    @property
    def out_dim(self):
        return self.layers[-1].w.shape[0]

    def param_arrays(self):
        return [a for l in self.layers for a in (l.w, l.b)]

    def copy(self):
        return Mlp([Layer(l.w.copy(), l.b.copy(), l.act) for l in self.layers])


class QuantizedMlp:
    """fp16 weights packed in access order (one neuron's row, then its bias)."""

    def __init__(self, shapes, acts, packed, clamped=0):
        self.shapes = [tuple(int(v) for v in s) for s in shapes]  # (out, in)
        self.acts = list(acts)
        self.packed = np.ascontiguousarray(packed, dtype=np.float16)
        self.clamped = int(clamped)
        need = sum(o * (i + 1) for o, i in self.shapes)
        if self.packed.size != need:
            raise ValueError("packed buffer size does not match the layer shapes")

    @property
    def in_dim(self):
        return self.shapes[0][1]

    @property
    def out_dim(self):
        return self.shapes[-1][0]

    def layer_views(self):
        """[(w fp32 (out,in), b fp32 (out,))] decoded from the packed buffer."""
        views, ofs = [], 0
        for out, fan_in in self.shapes:
            blk = self.packed[ofs:ofs + out * (fan_in + 1)].reshape(out, fan_in + 1)
            views.append((blk[:, :fan_in].astype(np.float32), blk[:, fan_in].astype(np.float32)))
            ofs += out * (fan_in + 1)
        return views

    def dequantize(self):
        return Mlp([Layer(w, b, a) for (w, b), a in zip(self.layer_views(), self.acts)])


def quantize(net):
    pieces, shapes, acts, clamped = [], [], [], 0
    for layer in net.layers:
        blk = np.concatenate([layer.w, layer.b[:, None]], axis=1)
        clamped += int(np.count_nonzero(np.abs(blk) > FP16_MAX))
        pieces.append(np.clip(blk, -FP16_MAX, FP16_MAX).astype(np.float16).ravel())
        shapes.append(layer.w.shape)
        acts.append(layer.act)
    return QuantizedMlp(shapes, acts, np.concatenate(pieces), clamped)


# --- NMWB0001 weight blob (f1: load trained reference materials) -------------

def write_blob(stream, net):
    q = quantize(net)
    stream.write(BLOB_MAGIC)
    stream.write(struct.pack("<I", len(net.layers)))
    for layer in net.layers:
        out, fan_in = layer.w.shape
        stream.write(struct.pack("<IIB", fan_in, out, ACT_CODES[layer.act]))
    for layer in net.layers:
        stream.write(layer.w.astype("<f4").tobytes())
        stream.write(layer.b.astype("<f4").tobytes())
    stream.write(q.packed.astype("<f2").tobytes())


def read_blob(stream):
    if stream.read(8) != BLOB_MAGIC:
        raise ValueError("not a weight blob")
    (n,) = struct.unpack("<I", stream.read(4))
    specs = [struct.unpack("<IIB", stream.read(9)) for _ in range(n)]
    layers = []
    for fan_in, out, act in specs:
        if act not in ACT_NAMES:
            raise ValueError("unknown activation code in blob")
        w = np.frombuffer(stream.read(4 * out * fan_in), dtype="<f4")
        b = np.frombuffer(stream.read(4 * out), dtype="<f4")
        if w.size != out * fan_in or b.size != out:
            raise ValueError("truncated weight blob")
        layers.append(Layer(w.reshape(out, fan_in), b, ACT_NAMES[act]))
    n_packed = sum((fi + 1) * o for fi, o, _ in specs)
    packed = np.frombuffer(stream.read(2 * n_packed), dtype="<f2")
    if packed.size != n_packed:
        raise ValueError("truncated weight blob")
    qnet = QuantizedMlp([(o, fi) for fi, o, _ in specs], [ACT_NAMES[a] for _, _, a in specs],
                        packed.astype(np.float16))
    return Mlp(layers), qnet


def blob_bytes(net):
    buf = io.BytesIO()
    write_blob(buf, net)
    return buf.getvalue()


def blob_from_bytes(data):
    return read_blob(io.BytesIO(data))
