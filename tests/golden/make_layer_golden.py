"""Golden fixtures for the layer around the hot path: the reference's layer_forward /
layer_backward (pkg/src/grkan/layer.py:318-379), y = W F(x) + bias and its gradients
(rational-stage bundle, d_weight and d_bias from the ascending row-block fold).

Imports the reference from /root/reference/pkg/src (build container only) and writes
tests/golden/layer_golden.npz + layer_golden.json; the fixtures travel, the reference
does not.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_layer_golden.py
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF_SRC)
    import grkan as g
    from grkan import layer as L

    arrays: dict[str, np.ndarray] = {}
    manifest = {"generator": "tests/golden/make_layer_golden.py", "numpy": np.__version__, "cases": {}}
    rng = np.random.default_rng(20250514)

    def case(name, batch, seq, d_in, d_out, groups, dtype, block, target=None, strategy=g.STRATEGY_BLOCKED,
             note=""):
        if target is None:  # random coefficients, as run_bench draws them
            params = g.GroupRationalParams(rng.standard_normal((groups, 6)), rng.standard_normal((groups, 4)))
            layer = L.GrKanLayer(params=params, layout=g.GroupLayout(d_in, groups),
                                 weight=rng.standard_normal((d_out, d_in)) / np.sqrt(d_in),
                                 bias=rng.standard_normal(d_out))
        else:  # make_layer's preset broadcast (layer.py:265-279)
            base = L.make_layer(d_in, d_out, groups, target=target,
                                weight=rng.standard_normal((d_out, d_in)) / np.sqrt(d_in))
            layer = L.GrKanLayer(params=base.params, layout=base.layout, weight=base.weight,
                                 bias=rng.standard_normal(d_out))
        x = g.ActivationTensor(rng.standard_normal((batch, seq, d_in)).astype(dtype))
        uy = g.ActivationTensor(rng.standard_normal((batch, seq, d_out)).astype(dtype))
        y = L.layer_forward(layer, x).data
        bundle, d_w, d_b = L.layer_backward(layer, x, uy, strategy=strategy, block_size=block)
        out = {"x": x.data, "uy": uy.data, "num": layer.params.numerator, "den": layer.params.denominator,
               "weight": layer.weight, "bias": layer.bias, "y": y, "d_x": bundle.d_x.data,
               "d_a": bundle.d_a, "d_b": bundle.d_b, "d_weight": d_w, "d_bias": d_b}
        for k, v in out.items():
            arrays["%s/%s" % (name, k)] = np.asarray(v)
        manifest["cases"][name] = {"shape": [batch, seq, d_in], "d_out": d_out, "groups": groups,
                                   "dtype": np.dtype(dtype).name, "block_size": block, "target": target,
                                   "strategy": strategy, "note": note}

    case("f32_swish_2x5x16_o8_g4", 2, 5, 16, 8, 4, np.float32, 4, target="swish",
         note="10 rows: row blocks 4, 4, 2 (ragged last block)")
    case("f64_swish_2x5x16_o8_g4", 2, 5, 16, 8, 4, np.float64, 4, target="swish")
    case("f32_identity_3x7x32_o16_g8", 3, 7, 32, 16, 8, np.float32, 8, target="identity",
         note="KAT's first rational is identity-initialised (A(x) = 0)")
    case("f32_gelu_2x9x64_o32_g8", 2, 9, 64, 32, 8, np.float32, 16, target="gelu")
    case("f32_random_4x33x64_o32_g8", 4, 33, 64, 32, 8, np.float32, 16, note="random coefficients, 132 rows")
    case("f64_random_3x11x48_o24_g4", 3, 11, 48, 24, 4, np.float64, 8)
    case("f32_swish_2x16x256_o64_g8", 2, 16, 256, 64, 8, np.float32, 8, target="swish",
         note="the fused tcgen05 layer's shape contract (d_in/groups = 32, d_out % 64 == 0)")
    case("f32_random_naive_2x6x32_o8_g4", 2, 6, 32, 8, 4, np.float32, 4, strategy=g.STRATEGY_NAIVE,
         note="layer_backward with the naive strategy")

    np.savez_compressed(os.path.join(HERE, "layer_golden.npz"), **arrays)
    with open(os.path.join(HERE, "layer_golden.json"), "w") as fh:
        json.dump(manifest, fh, indent=1, sort_keys=True)
    print("wrote %d arrays, %d cases" % (len(arrays), len(manifest["cases"])))


if __name__ == "__main__":
    main()
