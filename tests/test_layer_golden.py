"""The layer oracle (oracle/grkan_oracle.py layer_forward / layer_backward) pinned bit for
bit to the reference's own layer_forward / layer_backward outputs
(pkg/src/grkan/layer.py:318-379), recorded by tests/golden/make_layer_golden.py."""

import json
import os

import numpy as np
import pytest

from oracle import grkan_oracle as orc

HERE = os.path.dirname(os.path.abspath(__file__))


def layer_cases():
    with open(os.path.join(HERE, "golden", "layer_golden.json")) as fh:
        man = json.load(fh)
    z = np.load(os.path.join(HERE, "golden", "layer_golden.npz"))
    return [(name, meta, {k.split("/", 1)[1]: z[k] for k in z.files if k.startswith(name + "/")})
            for name, meta in sorted(man["cases"].items())]


@pytest.mark.parametrize("name,meta,arr", layer_cases(), ids=[c[0] for c in layer_cases()])
def test_layer_oracle_bitwise(name, meta, arr):
    y = orc.layer_forward(arr["x"], arr["num"], arr["den"], arr["weight"], arr["bias"])
    assert y.dtype == arr["y"].dtype and y.tobytes() == arr["y"].tobytes(), name
    dx, da, db, dw, dbias = orc.layer_backward(arr["x"], arr["uy"], arr["num"], arr["den"], arr["weight"],
                                               meta["block_size"], naive=meta["strategy"] == "naive_atomic")
    assert dx.tobytes() == arr["d_x"].tobytes(), name
    assert da.tobytes() == arr["d_a"].tobytes() and db.tobytes() == arr["d_b"].tobytes(), name
    assert dw.tobytes() == arr["d_weight"].tobytes() and dbias.tobytes() == arr["d_bias"].tobytes(), name
