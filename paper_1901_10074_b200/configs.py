"""Synthetic workloads of BASELINE.json's five configs.

No public dataset is involved: pixels and weights are drawn from
``numpy.random.default_rng(config number)`` in a fixed order (image, then
each layer's weights), keys and encryption randomness from
``default_rng(1234)`` shared by keygen and encryption (reference
cli.py:151-155).  The shapes are the configs' own.
"""

from __future__ import annotations

import numpy as np

from .inference import ConvSpec, FcSpec, NetworkSpec, SquareSpec
from .params import profile

KEY_SEED = 1234


def config_params(cfg: int):
    if cfg == 1:
        return profile("desk")
    if cfg in (2, 5):
        return profile("retina")
    if cfg == 3:
        # "modulus chain extended to the required depth": 24 x 30-bit q primes
        return profile("retina").replace(coeff_modulus_bits=720, name="retina-720")
    raise ValueError(f"no FV parameter set for config {cfg}")


def config_network(cfg: int, data_seed=None):
    """(image, NetworkSpec) of config 1, 2 (= 5 per image) or 3."""
    rng = np.random.default_rng(cfg if data_seed is None else data_seed)
    if cfg == 1:
        img = rng.integers(0, 256, (1, 16, 16), dtype=np.int64)
        conv = ConvSpec(2, (3, 3), (2, 2), (1, 16, 16), rng.integers(-4, 5, (2, 1, 3, 3)),
                        np.zeros(2, np.int64))
        fc = FcSpec(2, rng.integers(-4, 5, (2, conv.out_len)), np.zeros(2, np.int64))
        return img, NetworkSpec([conv, SquareSpec(), fc], (1, 16, 16))
    if cfg in (2, 5):
        img = rng.integers(0, 256, (1, 96, 96), dtype=np.int64)
        conv = ConvSpec(5, (5, 5), (2, 2), (1, 96, 96), rng.integers(-8, 9, (5, 1, 5, 5)),
                        np.zeros(5, np.int64))
        fc = FcSpec(2, rng.integers(-8, 9, (2, conv.out_len)), np.zeros(2, np.int64))
        return img, NetworkSpec([conv, SquareSpec(), fc], (1, 96, 96))
    if cfg == 3:
        img = rng.integers(0, 256, (3, 256, 256), dtype=np.int64)
        c1 = ConvSpec(8, (5, 5), (2, 2), (3, 256, 256), rng.integers(-8, 9, (8, 3, 5, 5)),
                      np.zeros(8, np.int64))
        c2 = ConvSpec(4, (3, 3), (2, 2), c1.out_shape, rng.integers(-8, 9, (4, 8, 3, 3)),
                      np.zeros(4, np.int64))
        fc = FcSpec(2, rng.integers(-8, 9, (2, c2.out_len)), np.zeros(2, np.int64))
        return img, NetworkSpec([c1, SquareSpec(), c2, SquareSpec(), fc], (3, 256, 256))
    raise ValueError(f"config {cfg} is not a network")


def batch_images(count: int = 256, seed: int = 5):
    """Config 5: ``count`` independent ROP-shaped images (weights of config 2)."""
    rng = np.random.default_rng(seed)
    return [rng.integers(0, 256, (1, 96, 96), dtype=np.int64) for _ in range(count)]


def plaintext_forward(net: NetworkSpec, img) -> list:
    """Exact Python-int forward pass (no int64 overflow): conv/fc/square."""
    x = np.asarray(img, dtype=object)
    for layer in net.layers:
        if isinstance(layer, SquareSpec):
            x = x * x
        elif isinstance(layer, ConvSpec):
            c, h, w = layer.in_shape
            kh, kw = layer.kernel
            sh, sw = layer.stride
            f, oh, ow = layer.out_shape
            xi = x.reshape(c, h, w)
            wts = np.asarray(layer.weights, dtype=object)
            out = np.empty((f, oh, ow), dtype=object)
            for fi in range(f):
                for oy in range(oh):
                    for ox in range(ow):
                        win = xi[:, oy * sh:oy * sh + kh, ox * sw:ox * sw + kw]
                        out[fi, oy, ox] = int((win * wts[fi]).sum()) + int(layer.biases[fi])
            x = out
        else:
            wm = np.asarray(layer.weights, dtype=object)
            x = wm.dot(x.reshape(-1)) + np.asarray(layer.biases, dtype=object)
    return [int(v) for v in np.asarray(x).reshape(-1)]


def centred_mod(values, t: int) -> list:
    out = []
    for v in values:
        r = int(v) % t
        out.append(r - t if r > t // 2 else r)
    return out


def workload_op_counts(cfg: int, data_seed=None) -> dict:
    """Exact serial op counts of one encrypted inference of a config
    (encryption of the input, every layer, decryption of the logits),
    computed on the host from the compiled layers -- no FV arithmetic."""
    from .inference import SquareSpec, compile_conv, compile_fc
    from .planner import count_layer_ops

    params = config_params(cfg)
    img, net = config_network(cfg, data_seed)
    s = params.slot_count
    pow2 = {1 << j for j in range((s - 1).bit_length())}
    length = int(np.prod(img.shape))
    k_cur = -(-length // s)
    tot = {"cmult": 0, "add": 0, "rotation": 0, "encrypt": k_cur, "mult": 0, "ks_hops": 0}
    for layer in net.layers:
        if isinstance(layer, SquareSpec):
            tot["mult"] += k_cur
            tot["ks_hops"] += k_cur  # one relinearisation per ct x ct product
            continue
        rows = compile_conv(layer, s) if isinstance(layer, ConvSpec) else compile_fc(layer, s)
        c = count_layer_ops(rows, k_cur, s, s, pow2)
        for key, v in c.items():
            tot[key] += v
        k_cur = max(1, -(-len(rows) // s))
    tot["decrypt"] = k_cur
    return tot
