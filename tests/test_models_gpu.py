"""GPU: the BASELINE model configs through the hot path.

* Node-by-node parity on reduced shapes: every node's GPU bound on the GPU's
  own node inputs vs the oracle op_bound on the same inputs
  (eps_ref <= eps_gpu <= eps_ref (1+1e-5)), values bit-exact where the
  reference defines them (sequential profile) -- ResNet (conv2d / BN / maxpool
  extensions) and GPT-2 (LayerNorm + affine, tanh-GELU, biases).
* Full-size configs (ResNet-18 B=32 224^2, GPT-2 small B=8 S=1024) run through
  the streaming verifier with one planted fault: exactly that node is flagged."""

import numpy as np
import pytest
import torch

from oracle import bounds as OB

pytestmark = pytest.mark.gpu
TRANSCENDENTAL = {"exp", "log", "tanh", "gelu", "silu"}


def _node_by_node(g, inputs, profile):
    from paper_2510_16028_b200.bounds import FpModel, op_bound_device
    from paper_2510_16028_b200.engine import to_device
    from paper_2510_16028_b200.graph import parse_ref
    model, values = FpModel(), {}
    for node in g.nodes:
        xs = []
        for ref in node.inputs:
            cat, key = parse_ref(ref)
            xs.append(values[key] if cat == "node" else to_device(
                inputs[key] if cat == "input" else g.weights[key]))
        y, eps = op_bound_device(node, xs, model, profile, eps_f64=True)
        values[node.index] = y
        if node.kind == "embedding":
            continue
        ins = [a.cpu().numpy() for a in xs]
        yr, ref = OB.op_bound(node, ins, OB.FpModel())
        y_h = y.cpu().numpy()
        if node.kind in ("matmul", "linear", "conv2d") and profile.reduction == "native":
            # native values come from cuBLAS/cuDNN (not a simulated profile): the bound
            # depends only on the inputs (+ u|y| on our own y for linear)
            if node.kind == "linear":
                ref = OB.matmul_bound(ins[0], ins[1], OB.FpModel()) + \
                    2.0 ** -24 * np.abs(y_h.astype(np.float64))
        elif node.kind not in TRANSCENDENTAL:
            assert np.array_equal(yr.view(np.uint32), y_h.view(np.uint32)), node.name
        e = eps.cpu().numpy()
        if node.kind in TRANSCENDENTAL:
            ref = 2 * 2.0 ** -24 * np.abs(y_h.astype(np.float64))
        assert np.all(e >= ref) and np.all(e <= ref * (1 + 1e-5) + 1e-300), node.name


@pytest.mark.parametrize("prof", ["sequential", "native"])
def test_resnet_small_node_by_node(prof):
    from paper_2510_16028_b200.engine import NATIVE, DeviceProfile
    from paper_2510_16028_b200.lowerings import build_resnet18
    from paper_2510_16028_b200.tensor import Rng
    torch.backends.cudnn.allow_tf32 = False
    spec = build_resnet18(batch=2, side=32, n_classes=10, width=8, seed=1)
    x = spec.make_inputs(Rng(3))
    _node_by_node(spec.graph, x, NATIVE if prof == "native" else DeviceProfile("s", "sequential"))


def test_gpt2_small_node_by_node():
    import dataclasses
    from paper_2510_16028_b200.engine import NATIVE
    from paper_2510_16028_b200.lowerings import GPT2_SMALL, build_decoder
    from paper_2510_16028_b200.tensor import Rng
    shape = dataclasses.replace(GPT2_SMALL, layers=2, hidden=64, heads=4, kv_heads=4,
                                head_dim=16, inter=256, vocab=300, seq=32, batch=2)
    spec = build_decoder(shape, seed=2)
    _node_by_node(spec.graph, spec.make_inputs(Rng(4)), NATIVE)


def _flagged(spec, fault):
    from paper_2510_16028_b200.dispute import CheckRecord
    from paper_2510_16028_b200.engine import NATIVE
    from paper_2510_16028_b200.executor import StreamingVerifier, drift_claim
    from paper_2510_16028_b200.tensor import Rng
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    sv = StreamingVerifier(spec.graph, None, NATIVE, None, "keccak256", 4096)
    roots, recs = sv.run(spec.make_inputs(Rng(5)),
                         lambda node, y: drift_claim(node, y, 3, 16, fault, 1e-2, 8))
    torch.cuda.synchronize()
    names = [n.name for n in spec.graph.nodes]
    return [names[i] for i in range(len(names)) if CheckRecord(recs[i]).host()["n_violations"]]


def test_resnet18_full_config_flags_only_the_fault():
    from paper_2510_16028_b200.lowerings import build_resnet18
    spec = build_resnet18(batch=32, side=224)
    assert _flagged(spec, "layer3.0.conv2") == ["layer3.0.conv2"]


def test_gpt2_small_full_config_flags_only_the_fault():
    from paper_2510_16028_b200.lowerings import GPT2_SMALL, build_decoder
    spec = build_decoder(GPT2_SMALL)
    assert _flagged(spec, "l5_fc") == ["l5_fc"]


def test_unet_small_node_by_node():
    from paper_2510_16028_b200.engine import NATIVE
    from paper_2510_16028_b200.lowerings import UNetShape, build_unet
    from paper_2510_16028_b200.tensor import Rng
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    shape = UNetShape(batch=1, latent=16, channels=(32, 64, 64, 64), heads=2, ctx_len=7,
                      ctx_dim=24, groups=8, temb=64)
    spec = build_unet(shape, seed=3)
    _node_by_node(spec.graph, spec.make_inputs(Rng(6)), NATIVE)


def test_unet_sd15_shape_flags_only_the_fault():
    """SD-1.5-shaped UNet at the BASELINE width (320/640/1280/1280, 8 heads,
    GroupNorm 32, 77x768 context) on a 32x32 latent, batch 1 (the 64x64 B=8
    config is the 8-GPU batch-sharded bench shape; per-sample work is the same graph)."""
    import dataclasses
    from paper_2510_16028_b200.lowerings import SD15_UNET, build_unet
    spec = build_unet(dataclasses.replace(SD15_UNET, batch=1, latent=32))
    assert _flagged(spec, "down1.res0.conv2") == ["down1.res0.conv2"]


def test_qwen3_8b_full_width_layers_flag_only_the_fault():
    """Two Qwen3-8B-shaped layers at full width and sequence (S=2048, H=4096,
    32/8 heads, I=12288) plus the LM head, through the streaming verifier with
    +-1-ulp drift on every reduction output: no bound violation anywhere but the
    node carrying the planted fault (BASELINE configs[3], bench.py's workload)."""
    import dataclasses
    from paper_2510_16028_b200.lowerings import QWEN3_8B, build_decoder
    spec = build_decoder(dataclasses.replace(QWEN3_8B, seq=2048), layers=2)
    assert _flagged(spec, "l1_down") == ["l1_down"]
