"""Graph lowerings of the BASELINE configs onto reference op kinds (+ the
"transpose" extension), so every node has a reference bound template.

* mlp      : the reference's own classifier graph (models.py:68-121) at the
             2-layer-MLP 784-256-10 B=64 config; same node list, names, attrs
             and Rng draws, so op signatures / weights are bit-identical
             (tests/test_lowerings.py checks the graph root against the golden).
* qwen3    : Qwen3-8B-shaped decoder (RMSNorm chains, q/k-norm, RoPE, GQA,
             eager causal attention, SiLU gate) -- SURVEY.md 2.3 lowering.
* gpt2     : GPT-2-small-shaped decoder (LayerNorm+affine, Conv1D linears,
             tanh-GELU, eager causal attention).
Weights for the large configs are generated on the GPU (torch, seeded):
random-init, synthetic -- the configs name shapes, not checkpoints.
"""

from __future__ import annotations

import math
import zlib
from dataclasses import dataclass, field

import numpy as np
import torch

from .graph import build_graph, input_ref, make_node, node_ref, weight_ref
from .tensor import Rng, Tensor


@dataclass
class ModelSpec:
    name: str
    graph: object
    input_kinds: dict
    n_classes: int = 0
    meta: dict = field(default_factory=dict)

    def make_inputs(self, rng: Rng) -> dict:
        """models.py:28-39."""
        out = {}
        for name, shape in self.graph.inputs:
            kind = self.input_kinds[name]
            if kind[0] == "uniform":
                out[name] = rng.uniform(shape, kind[1], kind[2])
            else:
                ids = rng.integers(0, kind[1], size=int(np.prod(shape)))
                out[name] = Tensor(shape, ids.astype(np.float32))
        return out


class _Builder:
    def __init__(self):
        self.nodes, self.weights = [], {}

    def add(self, name, kind, inputs, attrs=None) -> str:
        self.nodes.append(make_node(name, kind, inputs, attrs))
        return node_ref(len(self.nodes) - 1)

    def weight(self, name, rng: Rng, shape, lo, hi) -> str:
        self.weights[name] = rng.uniform(shape, lo, hi)
        return weight_ref(name)

    def tensor(self, name, t) -> str:
        self.weights[name] = t
        return weight_ref(name)


def build_mlp(seed: int = 0, batch: int = 64, in_dim: int = 784, hidden: int = 256,
              n_classes: int = 10) -> ModelSpec:
    """The reference MLP classifier graph (models.py:68-121): every
    non-embedding op kind; draws weights in the reference order."""
    rng = Rng(seed)
    b = _Builder()
    s = float(1.0 / np.sqrt(in_dim))
    W = lambda n, shp, lo, hi: b.weight(n, rng, shp, lo, hi)  # noqa: E731
    h = b.add("fc0", "linear", [input_ref("x"), W("w0", (in_dim, hidden), -s, s),
                                W("b0", (hidden,), -0.1, 0.1)])
    skip = h = b.add("act0", "gelu", [h])
    h = b.add("fc1", "linear", [h, W("w1", (hidden, hidden), -0.2, 0.2),
                                W("b1", (hidden,), -0.1, 0.1)])
    h = b.add("res1", "add", [h, skip])
    h = b.add("ln1", "layernorm", [h], {"axis": -1, "eps": 1e-5})
    h = b.add("act1", "relu", [h])
    h = b.add("mm1", "matmul", [h, W("w2", (hidden, hidden), -0.2, 0.2)])
    h = b.add("act2", "tanh", [h])
    h = b.add("scale1", "mul", [h, W("wm", (hidden,), 0.5, 1.5)])
    h = b.add("shift1", "sub", [h, W("wb", (hidden,), -0.2, 0.2)])
    h = b.add("neg1", "neg", [h])
    h = b.add("act3", "silu", [h])
    mx = b.add("rowmax", "max", [h], {"axis": 1})
    mxc = b.add("rowmax_col", "reshape", [mx], {"shape": f"{batch},1"})
    h2 = b.add("center", "sub", [h, mxc])
    eh = b.add("expo", "exp", [h2])
    sm = b.add("rowsum", "sum", [eh], {"axis": 1})
    smc = b.add("rowsum_col", "reshape", [sm], {"shape": f"{batch},1"})
    p = b.add("norm", "div", [eh, smc])
    sq = b.add("square", "mul", [p, p])
    pos = b.add("lift", "add", [sq, W("wc", (hidden,), 0.8, 1.2)])
    rt = b.add("root", "sqrt", [pos])
    irt = b.add("invroot", "rsqrt", [pos])
    mixed = b.add("mix", "add", [rt, irt])
    lg = b.add("logpos", "log", [pos])
    cat = b.add("widen", "concat", [mixed, lg], {"axis": 1})
    cut = b.add("window", "slice", [cat], {"axis": 1, "start": hidden // 2,
                                           "stop": hidden // 2 + hidden})
    mu = b.add("rowmean", "mean", [cut], {"axis": 1})
    mn = b.add("rowmin", "min", [cut], {"axis": 1})
    spread = b.add("spread", "sub", [mu, mn])
    spreadc = b.add("spread_col", "reshape", [spread], {"shape": f"{batch},1"})
    h3 = b.add("recenter", "add", [cut, spreadc])
    h3 = b.add("ln2", "layernorm", [h3], {"axis": -1, "eps": 1e-5})
    h3 = b.add("attend", "softmax", [h3], {"axis": -1})
    logits = b.add("head", "linear", [h3, W("w3", (hidden, n_classes), -0.4, 0.4),
                                      W("b3", (n_classes,), 1.5, 2.5)])
    g = build_graph(b.nodes, [("x", (batch, in_dim))], b.weights, [logits])
    return ModelSpec("mlp", g, {"x": ("uniform", -1.0, 1.0)}, n_classes)


# --------------------------------------------------------------- decoders

@dataclass(frozen=True)
class DecoderShape:
    name: str
    layers: int
    hidden: int
    heads: int
    kv_heads: int
    head_dim: int
    inter: int
    vocab: int
    seq: int
    batch: int = 1
    norm: str = "rms"          # "rms" (Qwen3) | "ln" (GPT-2)
    qk_norm: bool = True
    rope: bool = True
    act: str = "silu_gate"     # "silu_gate" | "gelu"
    bias: bool = False
    eps: float = 1e-6


QWEN3_8B = DecoderShape("qwen3-8b", layers=36, hidden=4096, heads=32, kv_heads=8, head_dim=128,
                        inter=12288, vocab=151936, seq=2048)
GPT2_SMALL = DecoderShape("gpt2-small", layers=12, hidden=768, heads=12, kv_heads=12, head_dim=64,
                          inter=3072, vocab=50257, seq=1024, batch=8, norm="ln", qk_norm=False,
                          rope=False, act="gelu", bias=True, eps=1e-5)


class _LazyWeights(dict):
    """name -> Tensor generated on first access on the GPU (seeded per name)."""

    def __init__(self, specs: dict, device: str, seed: int):
        super().__init__()
        self.specs, self.device, self.seed = specs, device, seed

    def __contains__(self, k):
        return k in self.specs

    def shape_of(self, k) -> tuple:
        """Shape without materialising the weight."""
        return tuple(self.specs[k][0])

    def __missing__(self, k):
        shape, kind, a = self.specs[k]
        gen = torch.Generator(device=self.device)
        gen.manual_seed(zlib.crc32(f"{self.seed}:{k}".encode()))
        if kind == "uniform":
            t = (torch.rand(shape, generator=gen, device=self.device) * 2 - 1) * a
        elif kind == "normal":
            t = torch.randn(shape, generator=gen, device=self.device) * a
        elif kind == "const":
            t = torch.as_tensor(a, dtype=torch.float32, device=self.device).reshape(shape)
        else:
            t = a(shape)
        t = t.float().contiguous()
        v = Tensor(shape, t)
        dict.__setitem__(self, k, v)
        return v

    def __iter__(self):
        return iter(self.specs)

    def __len__(self):
        return len(self.specs)

    def keys(self):
        return self.specs.keys()

    def items(self):
        return ((k, self[k]) for k in self.specs)


def _rope_tables(seq: int, dim: int, theta: float = 1_000_000.0):
    inv = 1.0 / (theta ** (np.arange(0, dim, 2, dtype=np.float64) / dim))
    ang = np.outer(np.arange(seq, dtype=np.float64), inv)
    emb = np.concatenate([ang, ang], axis=-1)
    return np.cos(emb).astype(np.float32), np.sin(emb).astype(np.float32)


def build_decoder(shape: DecoderShape, device: str = "cuda", seed: int = 0,
                  layers: int | None = None, with_head: bool = True) -> ModelSpec:
    """Eager decoder lowered onto reference kinds.  Node list per layer:
    norm chain, q/k/v projections, (q/k RMSNorm), RoPE (slice/neg/concat/mul/add),
    GQA expansion (reshape/concat), scores (matmul transpose_b), scale (mul),
    causal mask (add, finite -1e9), softmax, context matmul, out projection,
    residual add, MLP (SiLU-gate or GELU), residual add."""
    L = shape.layers if layers is None else layers
    H, nh, nkv, hd, I = shape.hidden, shape.heads, shape.kv_heads, shape.head_dim, shape.inter
    S, B = shape.seq, shape.batch
    T = B * S
    specs = {}
    nodes = []

    def add(name, kind, inputs, attrs=None):
        nodes.append(make_node(name, kind, inputs, attrs))
        return node_ref(len(nodes) - 1)

    def W(name, shp, kind="uniform", a=None):
        if a is None:
            a = 1.0 / math.sqrt(shp[0])
        specs[name] = (tuple(shp), kind, a)
        return weight_ref(name)

    def norm(prefix, x, width, rows_shape):
        """RMSNorm: sq, mean, +eps, rsqrt, reshape, mul, mul(weight) -- or LayerNorm(+affine)."""
        if shape.norm == "ln":
            y = add(f"{prefix}_ln", "layernorm", [x], {"axis": -1, "eps": shape.eps})
            y = add(f"{prefix}_g", "mul", [y, W(f"{prefix}.g", (width,), "uniform", 1.0)])
            return add(f"{prefix}_b", "add", [y, W(f"{prefix}.b", (width,), "uniform", 0.1)])
        sq = add(f"{prefix}_sq", "mul", [x, x])
        ms = add(f"{prefix}_ms", "mean", [sq], {"axis": -1})
        mse = add(f"{prefix}_mse", "add", [ms, W(f"{prefix}.eps", (1,), "const",
                                                  [shape.eps])])
        r = add(f"{prefix}_r", "rsqrt", [mse])
        rc = add(f"{prefix}_rc", "reshape", [r], {"shape": ",".join(map(str, rows_shape + (1,)))})
        xn = add(f"{prefix}_xn", "mul", [x, rc])
        return add(f"{prefix}_w", "mul", [xn, W(f"{prefix}.w", (width,), "uniform", 1.0)])

    x = add("embed", "embedding", [input_ref("ids"), W("embed.w", (shape.vocab, H), "normal", 0.02)])
    if shape.norm == "ln":
        x = add("posadd", "add", [x, W("pos.w", (S, H), "normal", 0.01)])
    x = add("flatten", "reshape", [x], {"shape": f"{T},{H}"})
    cos, sin = _rope_tables(S, hd)
    if shape.rope:
        specs["rope.cos"] = ((1, S, hd), "const", cos.reshape(-1))
        specs["rope.sin"] = ((1, S, hd), "const", sin.reshape(-1))
    mask = np.triu(np.full((S, S), -1e9, dtype=np.float32), k=1)
    specs["attn.mask"] = ((S, S), "const", mask.reshape(-1))
    specs["attn.scale"] = ((1,), "const", [1.0 / math.sqrt(hd)])

    for l in range(L):
        p = f"l{l}"
        h_in = x
        xn = norm(f"{p}_in", x, H, (T,))

        def proj(name, inp, k_in, n_out):
            y = add(f"{p}_{name}", "matmul", [inp, W(f"{p}.{name}.w", (k_in, n_out))])
            if shape.bias:
                y = add(f"{p}_{name}_bias", "add", [y, W(f"{p}.{name}.b", (n_out,), "uniform", 0.02)])
            return y

        q = proj("q", xn, H, nh * hd)
        k = proj("k", xn, H, nkv * hd)
        v = proj("v", xn, H, nkv * hd)
        # heads: [B,S,h,hd] -> [B,h,S,hd] (flattened batch*heads)
        q = add(f"{p}_q4", "reshape", [q], {"shape": f"{B},{S},{nh},{hd}"})
        k = add(f"{p}_k4", "reshape", [k], {"shape": f"{B},{S},{nkv},{hd}"})
        v = add(f"{p}_v4", "reshape", [v], {"shape": f"{B},{S},{nkv},{hd}"})
        if shape.qk_norm:
            q = norm(f"{p}_qn", q, hd, (B, S, nh))
            k = norm(f"{p}_kn", k, hd, (B, S, nkv))
        q = add(f"{p}_qt", "transpose", [q], {"perm": "0,2,1,3"})
        k = add(f"{p}_kt", "transpose", [k], {"perm": "0,2,1,3"})
        v = add(f"{p}_vt", "transpose", [v], {"perm": "0,2,1,3"})
        if shape.rope:
            def rope(tag, t, nheads):
                t3 = add(f"{p}_{tag}3", "reshape", [t], {"shape": f"{B * nheads},{S},{hd}"})
                lo = add(f"{p}_{tag}lo", "slice", [t3], {"axis": -1, "start": 0, "stop": hd // 2})
                hi = add(f"{p}_{tag}hi", "slice", [t3], {"axis": -1, "start": hd // 2, "stop": hd})
                nhi = add(f"{p}_{tag}nhi", "neg", [hi])
                rot = add(f"{p}_{tag}rot", "concat", [nhi, lo], {"axis": -1})
                c = add(f"{p}_{tag}cos", "mul", [t3, weight_ref("rope.cos")])
                s_ = add(f"{p}_{tag}sin", "mul", [rot, weight_ref("rope.sin")])
                return add(f"{p}_{tag}rope", "add", [c, s_])
            q = rope("q", q, nh)
            k = rope("k", k, nkv)
        else:
            q = add(f"{p}_q3", "reshape", [q], {"shape": f"{B * nh},{S},{hd}"})
            k = add(f"{p}_k3", "reshape", [k], {"shape": f"{B * nkv},{S},{hd}"})
        v = add(f"{p}_v3", "reshape", [v], {"shape": f"{B * nkv},{S},{hd}"})
        if nkv != nh:  # GQA: kv head j serves q heads j*g .. j*g+g-1
            grp = nh // nkv
            k = add(f"{p}_k5", "reshape", [k], {"shape": f"{B * nkv},1,{S},{hd}"})
            v = add(f"{p}_v5", "reshape", [v], {"shape": f"{B * nkv},1,{S},{hd}"})
            k = add(f"{p}_kx", "concat", [k] * grp, {"axis": 1})
            v = add(f"{p}_vx", "concat", [v] * grp, {"axis": 1})
            k = add(f"{p}_kg", "reshape", [k], {"shape": f"{B * nh},{S},{hd}"})
            v = add(f"{p}_vg", "reshape", [v], {"shape": f"{B * nh},{S},{hd}"})
        sc = add(f"{p}_scores", "matmul", [q, k], {"transpose_b": 1})
        sc = add(f"{p}_scaled", "mul", [sc, weight_ref("attn.scale")])
        sc = add(f"{p}_masked", "add", [sc, weight_ref("attn.mask")])
        pr = add(f"{p}_probs", "softmax", [sc], {"axis": -1})
        ctx = add(f"{p}_ctx", "matmul", [pr, v])
        ctx = add(f"{p}_ctx4", "reshape", [ctx], {"shape": f"{B},{nh},{S},{hd}"})
        ctx = add(f"{p}_ctxt", "transpose", [ctx], {"perm": "0,2,1,3"})
        ctx = add(f"{p}_ctx2", "reshape", [ctx], {"shape": f"{T},{nh * hd}"})
        o = proj("o", ctx, nh * hd, H)
        x = add(f"{p}_res1", "add", [h_in, o])
        xn2 = norm(f"{p}_post", x, H, (T,))
        if shape.act == "silu_gate":
            gt = proj("gate", xn2, H, I)
            up = proj("up", xn2, H, I)
            ga = add(f"{p}_act", "silu", [gt])
            hh = add(f"{p}_glu", "mul", [ga, up])
        else:
            up = proj("fc", xn2, H, I)
            hh = add(f"{p}_act", "gelu", [up])
        dn = proj("down", hh, I, H)
        x = add(f"{p}_res2", "add", [x, dn])
    x = norm("final", x, H, (T,))
    out = x
    if with_head:
        out = add("lm_head", "matmul", [x, W("lm_head.w", (H, shape.vocab))])
    weights = _LazyWeights(specs, device, seed)
    g = build_graph(nodes, [("ids", (B, S))], weights, [out])
    return ModelSpec(shape.name, g, {"ids": ("tokens", shape.vocab)},
                     meta={"shape": shape, "layers": L})


# --------------------------------------------------------------- ResNet-18

def build_resnet18(batch: int = 32, side: int = 224, n_classes: int = 1000, width: int = 64,
                   device: str = "cuda", seed: int = 0) -> ModelSpec:
    """ResNet-18 (eval) lowered onto reference kinds + conv2d / maxpool2d
    extensions: conv -> BN as sub / mul / add with per-channel
    constants (single-rounding templates) -> relu; maxpool; global average
    pool = reshape + mean; fc = linear.  Kaiming-normal convs, randomised BN
    running statistics, images U(-1, 1) (BASELINE config 2)."""
    specs, nodes = {}, []

    def add(name, kind, inputs, attrs=None):
        nodes.append(make_node(name, kind, inputs, attrs))
        return node_ref(len(nodes) - 1)

    def conv(name, x, cin, cout, k, stride, pad):
        specs[f"{name}.w"] = ((cout, cin, k, k), "normal", math.sqrt(2.0 / (cin * k * k)))
        return add(name, "conv2d", [x, weight_ref(f"{name}.w")], {"stride": stride, "pad": pad})

    def bn(name, x, c):
        rng = np.random.default_rng(zlib.crc32(name.encode()) + seed)
        mean = rng.uniform(-0.1, 0.1, c)
        var = rng.uniform(0.5, 1.5, c)
        gamma = rng.uniform(0.8, 1.2, c)
        beta = rng.uniform(-0.1, 0.1, c)
        scale = (gamma / np.sqrt(var + 1e-5)).astype(np.float32)
        specs[f"{name}.mean"] = ((1, c, 1, 1), "const", mean.astype(np.float32))
        specs[f"{name}.scale"] = ((1, c, 1, 1), "const", scale)
        specs[f"{name}.beta"] = ((1, c, 1, 1), "const", beta.astype(np.float32))
        y = add(f"{name}_sub", "sub", [x, weight_ref(f"{name}.mean")])
        y = add(f"{name}_mul", "mul", [y, weight_ref(f"{name}.scale")])
        return add(f"{name}_add", "add", [y, weight_ref(f"{name}.beta")])

    x = input_ref("img")
    h = conv("conv1", x, 3, width, 7, 2, 3)
    h = bn("bn1", h, width)
    h = add("relu1", "relu", [h])
    h = add("maxpool", "maxpool2d", [h], {"k": 3, "stride": 2, "pad": 1})
    cin, sp = width, side // 4
    for li, (cout, stride) in enumerate([(width, 1), (2 * width, 2), (4 * width, 2),
                                         (8 * width, 2)]):
        for bi in range(2):
            p = f"layer{li + 1}.{bi}"
            s = stride if bi == 0 else 1
            idn = h
            y = conv(f"{p}.conv1", h, cin, cout, 3, s, 1)
            y = bn(f"{p}.bn1", y, cout)
            y = add(f"{p}.relu1", "relu", [y])
            y = conv(f"{p}.conv2", y, cout, cout, 3, 1, 1)
            y = bn(f"{p}.bn2", y, cout)
            if s != 1 or cin != cout:
                idn = conv(f"{p}.down", h, cin, cout, 1, s, 0)
                idn = bn(f"{p}.downbn", idn, cout)
            y = add(f"{p}.res", "add", [y, idn])
            h = add(f"{p}.relu2", "relu", [y])
            cin = cout
        sp = sp if li == 0 else sp // 2
    h = add("pool_flat", "reshape", [h], {"shape": f"{batch},{cin},{sp * sp}"})
    h = add("avgpool", "mean", [h], {"axis": -1})
    specs["fc.w"] = ((cin, n_classes), "uniform", 1.0 / math.sqrt(cin))
    specs["fc.b"] = ((n_classes,), "uniform", 1.0 / math.sqrt(cin))
    out = add("fc", "linear", [h, weight_ref("fc.w"), weight_ref("fc.b")])
    g = build_graph(nodes, [("img", (batch, 3, side, side))], _LazyWeights(specs, device, seed),
                    [out])
    return ModelSpec("resnet18", g, {"img": ("uniform", -1.0, 1.0)}, n_classes)


# ------------------------------------------------------------ SD-UNet

@dataclass(frozen=True)
class UNetShape:
    name: str = "sd15-unet"
    batch: int = 8
    latent: int = 64
    in_ch: int = 4
    channels: tuple = (320, 640, 1280, 1280)
    attn_levels: tuple = (True, True, True, False)
    heads: int = 8
    ctx_len: int = 77
    ctx_dim: int = 768
    groups: int = 32
    temb: int = 1280
    layers_per_block: int = 2


SD15_UNET = UNetShape()


def build_unet(shape: UNetShape = SD15_UNET, device: str = "cuda", seed: int = 0) -> ModelSpec:
    """SD-1.5-shaped UNet denoising step (BASELINE config 5) on reference kinds
    + conv2d / upsample2x extensions: GroupNorm = reshape + layernorm + reshape +
    mul + add; SiLU; ResBlocks with the time-embedding projection broadcast-added;
    transformer blocks (LayerNorm, self-attention, cross-attention to the text
    context, tanh-GELU GEGLU feed-forward); skip concats; nearest 2x upsampling.
    The sinusoidal timestep embedding (t = 500) is a constant input feature."""
    B, C0 = shape.batch, shape.channels[0]
    specs, nodes = {}, []

    def add(name, kind, inputs, attrs=None):
        nodes.append(make_node(name, kind, inputs, attrs))
        return node_ref(len(nodes) - 1)

    def W(name, shp, kind="uniform", a=None):
        if a is None:
            fan = int(np.prod(shp[1:])) if len(shp) == 4 else shp[0]
            a = 1.0 / math.sqrt(fan)
        specs[name] = (tuple(shp), kind, a)
        return weight_ref(name)

    def conv(name, x, cin, cout, k=3, stride=1):
        y = add(name, "conv2d", [x, W(f"{name}.w", (cout, cin, k, k))],
                {"stride": stride, "pad": k // 2})
        return add(f"{name}_b", "add", [y, W(f"{name}.b", (1, cout, 1, 1), "uniform", 0.02)])

    def groupnorm(name, x, c, hw):
        g = shape.groups
        y = add(f"{name}_g", "reshape", [x], {"shape": f"{B},{g},{(c // g) * hw}"})
        y = add(f"{name}_ln", "layernorm", [y], {"axis": -1, "eps": 1e-5})
        y = add(f"{name}_r", "reshape", [y], {"shape": f"{B},{c},{int(math.isqrt(hw))},{int(math.isqrt(hw))}"})
        y = add(f"{name}_s", "mul", [y, W(f"{name}.g", (1, c, 1, 1), "uniform", 1.0)])
        return add(f"{name}_t", "add", [y, W(f"{name}.bt", (1, c, 1, 1), "uniform", 0.1)])

    def resblock(name, x, cin, cout, side, temb):
        h = groupnorm(f"{name}.gn1", x, cin, side * side)
        h = add(f"{name}.act1", "silu", [h])
        h = conv(f"{name}.conv1", h, cin, cout)
        t = add(f"{name}.tact", "silu", [temb])
        t = add(f"{name}.tproj", "linear", [t, W(f"{name}.tw", (shape.temb, cout)),
                                           W(f"{name}.tb", (cout,), "uniform", 0.02)])
        t = add(f"{name}.t4", "reshape", [t], {"shape": f"{B},{cout},1,1"})
        h = add(f"{name}.tadd", "add", [h, t])
        h = groupnorm(f"{name}.gn2", h, cout, side * side)
        h = add(f"{name}.act2", "silu", [h])
        h = conv(f"{name}.conv2", h, cout, cout)
        skip = x if cin == cout else conv(f"{name}.skip", x, cin, cout, k=1)
        return add(f"{name}.res", "add", [h, skip])

    def attention(name, xq, xkv, c, n_q, n_kv, kv_dim):
        hd = c // shape.heads
        q = add(f"{name}.q", "matmul", [xq, W(f"{name}.wq", (c, c))])
        k = add(f"{name}.k", "matmul", [xkv, W(f"{name}.wk", (kv_dim, c))])
        v = add(f"{name}.v", "matmul", [xkv, W(f"{name}.wv", (kv_dim, c))])
        q = add(f"{name}.q4", "reshape", [q], {"shape": f"{B},{n_q},{shape.heads},{hd}"})
        k = add(f"{name}.k4", "reshape", [k], {"shape": f"{B},{n_kv},{shape.heads},{hd}"})
        v = add(f"{name}.v4", "reshape", [v], {"shape": f"{B},{n_kv},{shape.heads},{hd}"})
        q = add(f"{name}.qt", "transpose", [q], {"perm": "0,2,1,3"})
        k = add(f"{name}.kt", "transpose", [k], {"perm": "0,2,1,3"})
        v = add(f"{name}.vt", "transpose", [v], {"perm": "0,2,1,3"})
        s = add(f"{name}.scores", "matmul", [q, k], {"transpose_b": 1})
        s = add(f"{name}.scaled", "mul", [s, W(f"{name}.scale", (1,), "const", [1.0 / math.sqrt(hd)])])
        p = add(f"{name}.probs", "softmax", [s], {"axis": -1})
        o = add(f"{name}.ctx", "matmul", [p, v])
        o = add(f"{name}.ctxt", "transpose", [o], {"perm": "0,2,1,3"})
        o = add(f"{name}.ctx2", "reshape", [o], {"shape": f"{B},{n_q},{c}"})
        o = add(f"{name}.o", "matmul", [o, W(f"{name}.wo", (c, c))])
        return add(f"{name}.ob", "add", [o, W(f"{name}.bo", (c,), "uniform", 0.02)])

    def transformer(name, x, c, side):
        n = side * side
        h = groupnorm(f"{name}.gn", x, c, n)
        h = add(f"{name}.flat", "reshape", [h], {"shape": f"{B},{c},{n}"})
        h = add(f"{name}.tok", "transpose", [h], {"perm": "0,2,1"})
        h = add(f"{name}.pin", "matmul", [h, W(f"{name}.pin.w", (c, c))])
        a = add(f"{name}.ln1", "layernorm", [h], {"axis": -1, "eps": 1e-5})
        h = add(f"{name}.r1", "add", [h, attention(f"{name}.sa", a, a, c, n, n, c)])
        a = add(f"{name}.ln2", "layernorm", [h], {"axis": -1, "eps": 1e-5})
        h = add(f"{name}.r2", "add", [h, attention(f"{name}.ca", a, input_ref("context"), c, n,
                                                     shape.ctx_len, shape.ctx_dim)])
        a = add(f"{name}.ln3", "layernorm", [h], {"axis": -1, "eps": 1e-5})
        ff = add(f"{name}.ff1", "linear", [a, W(f"{name}.ff1.w", (c, 8 * c)),
                                          W(f"{name}.ff1.b", (8 * c,), "uniform", 0.02)])
        xg = add(f"{name}.ffx", "slice", [ff], {"axis": -1, "start": 0, "stop": 4 * c})
        gt = add(f"{name}.ffg", "slice", [ff], {"axis": -1, "start": 4 * c, "stop": 8 * c})
        gt = add(f"{name}.ffact", "gelu", [gt])
        ff = add(f"{name}.geglu", "mul", [xg, gt])
        ff = add(f"{name}.ff2", "linear", [ff, W(f"{name}.ff2.w", (4 * c, c)),
                                          W(f"{name}.ff2.b", (c,), "uniform", 0.02)])
        h = add(f"{name}.r3", "add", [h, ff])
        h = add(f"{name}.pout", "matmul", [h, W(f"{name}.pout.w", (c, c))])
        h = add(f"{name}.untok", "transpose", [h], {"perm": "0,2,1"})
        h = add(f"{name}.unflat", "reshape", [h], {"shape": f"{B},{c},{side},{side}"})
        return add(f"{name}.res", "add", [h, x])

    # timestep embedding: sinusoid(t) is a constant feature, then MLP
    half = C0 // 2
    freqs = np.exp(-math.log(10000.0) * np.arange(half) / half)
    sin = np.concatenate([np.cos(500.0 * freqs), np.sin(500.0 * freqs)]).astype(np.float32)
    specs["tsin"] = ((B, C0), "const", np.tile(sin, B))
    temb = add("temb1", "linear", [weight_ref("tsin"), W("temb1.w", (C0, shape.temb)),
                                   W("temb1.b", (shape.temb,), "uniform", 0.02)])
    temb = add("temb_act", "silu", [temb])
    temb = add("temb2", "linear", [temb, W("temb2.w", (shape.temb, shape.temb)),
                                   W("temb2.b", (shape.temb,), "uniform", 0.02)])
    h = conv("conv_in", input_ref("latent"), shape.in_ch, C0)
    side, cin = shape.latent, C0
    skips = [(h, cin, side)]
    for lvl, (c, attn) in enumerate(zip(shape.channels, shape.attn_levels)):
        for j in range(shape.layers_per_block):
            h = resblock(f"down{lvl}.res{j}", h, cin, c, side, temb)
            cin = c
            if attn:
                h = transformer(f"down{lvl}.tf{j}", h, c, side)
            skips.append((h, c, side))
        if lvl < len(shape.channels) - 1:
            h = conv(f"down{lvl}.ds", h, c, c, k=3, stride=2)
            side //= 2
            skips.append((h, c, side))
    c = shape.channels[-1]
    h = resblock("mid.res0", h, c, c, side, temb)
    h = transformer("mid.tf", h, c, side)
    h = resblock("mid.res1", h, c, c, side, temb)
    for lvl in reversed(range(len(shape.channels))):
        c = shape.channels[lvl]
        for j in range(shape.layers_per_block + 1):
            s_ref, s_c, _ = skips.pop()
            h = add(f"up{lvl}.cat{j}", "concat", [h, s_ref], {"axis": 1})
            h = resblock(f"up{lvl}.res{j}", h, cin + s_c, c, side, temb)
            cin = c
            if shape.attn_levels[lvl]:
                h = transformer(f"up{lvl}.tf{j}", h, c, side)
        if lvl > 0:
            h = add(f"up{lvl}.us", "upsample2x", [h])
            side *= 2
            h = conv(f"up{lvl}.usconv", h, c, c)
    h = groupnorm("out.gn", h, cin, side * side)
    h = add("out.act", "silu", [h])
    out = conv("conv_out", h, cin, shape.in_ch)
    weights = _LazyWeights(specs, device, seed)
    g = build_graph(nodes, [("latent", (B, shape.in_ch, shape.latent, shape.latent)),
                            ("context", (B, shape.ctx_len, shape.ctx_dim))], weights, [out])
    return ModelSpec(shape.name, g, {"latent": ("uniform", -1.0, 1.0),
                                     "context": ("uniform", -1.0, 1.0)}, meta={"shape": shape})
