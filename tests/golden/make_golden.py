"""Generate the golden fixtures that pin the oracle (and, through it, the GPU path).

This script imports the *reference* package (``grkan``) from
``/root/reference/pkg/src`` and records its outputs on seeded inputs.  It runs
only in the build container (the reference is not present on the GPU box); the
committed ``grkan_golden.npz`` + ``grkan_golden.json`` travel instead.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Every case records the inputs (or, for the KAT-T case, the seed that
regenerates them with ``run_bench``'s draw order, pkg/src/grkan/cli.py:146-158),
the reference forward (``forward_tensor``, pkg/src/grkan/rational.py:325), both
backward strategies (``backward_blocked`` pkg/src/grkan/backward.py:275 and
``backward_naive`` :187), the fp64 accumulation of the run-precision terms
(``reference_coeff_grads``, pkg/src/grkan/verification.py:318) and, for small
cases, the triple-loop fp64 oracle (``oracle_backward``, verification.py:49).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _import_reference():
    sys.dont_write_bytecode = True
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import grkan  # noqa: F401
    from grkan import verification  # noqa: F401
    return grkan


def sha(arr: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def kat_t_inputs(seed=0, batch=8, seq=197, dim=192, groups=8, m1=6, n=4, dtype=np.float32):
    """run_bench's exact draw order (pkg/src/grkan/cli.py:146-158)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((batch, seq, dim)).astype(dtype)
    u = rng.standard_normal((batch, seq, dim)).astype(dtype)
    num = rng.standard_normal((groups, m1))
    den = rng.standard_normal((groups, n))
    return x, u, num, den


def main():
    g = _import_reference()
    from grkan.verification import oracle_backward, reference_coeff_grads
    from grkan.layer import load_builtin_preset

    arrays: dict[str, np.ndarray] = {}
    manifest: dict = {"generator": "tests/golden/make_golden.py", "numpy": np.__version__,
                      "cases": {}, "scalars": [], "presets": {}}

    def run_case(name, x, u, num, den, groups, block, store_inputs=True, store_outputs=True,
                 with_oracle=False, note=""):
        layout = g.GroupLayout(x.shape[2], groups)
        params = g.GroupRationalParams(num, den)
        xt = g.ActivationTensor(x)
        ut = g.ActivationTensor(u)
        y = g.forward_tensor(xt, params, layout, validate=False).data
        plan = g.ExecutionPlan.blocked(x.shape[0], x.shape[1], layout, block)
        meta = {"shape": list(x.shape), "dtype": str(x.dtype), "groups": groups,
                "m1": int(params.num_coeffs), "n": int(params.den_coeffs),
                "block_size": block, "note": note, "error": None}
        try:
            with np.errstate(over="ignore", invalid="ignore"):
                blk = g.backward_blocked(xt, ut, params, plan, validate=False)
        except g.GrkanError as exc:  # recorded as the expected error class
            meta["error"] = type(exc).__name__
            blk = None
        try:
            with np.errstate(over="ignore", invalid="ignore"):
                nav = g.backward_naive(xt, ut, params, validate=False)
        except g.GrkanError as exc:
            meta["error_naive"] = type(exc).__name__
            nav = None
        with np.errstate(over="ignore", invalid="ignore"):
            ref_a, ref_b = reference_coeff_grads(xt, ut, params, layout)
        out = {"num": params.numerator, "den": params.denominator, "ref64_da": ref_a,
               "ref64_db": ref_b}
        if store_inputs:
            out["x"] = x
            out["u"] = u
        meta["sha_y"] = sha(y)
        if blk is not None:
            out["blocked_da"] = blk.d_a
            out["blocked_db"] = blk.d_b
            meta["sha_dx"] = sha(blk.d_x.data)
        if nav is not None:
            out["naive_da"] = nav.d_a
            out["naive_db"] = nav.d_b
            meta["sha_dx_naive"] = sha(nav.d_x.data)
        if store_outputs:
            out["y"] = y
            if blk is not None:
                out["dx"] = blk.d_x.data
        else:
            # strided samples for debugging a hash mismatch
            flat_idx = np.linspace(0, y.size - 1, 4096).astype(np.int64)
            out["sample_idx"] = flat_idx
            out["sample_y"] = y.reshape(-1)[flat_idx]
            if blk is not None:
                out["sample_dx"] = blk.d_x.data.reshape(-1)[flat_idx]
        if with_oracle:
            orc = oracle_backward(xt, ut, params, layout)
            out["oracle_da"] = orc.d_a
            out["oracle_db"] = orc.d_b
            out["oracle_dx"] = orc.d_x.data
        for k, v in out.items():
            arrays["%s/%s" % (name, k)] = np.asarray(v)
        manifest["cases"][name] = meta

    rng = np.random.default_rng(20250513)

    def rnd(shape, groups, m1=6, n=4, dtype=np.float32, scale=1.0):
        x = (rng.standard_normal(shape) * scale).astype(dtype)
        u = rng.standard_normal(shape).astype(dtype)
        num = rng.standard_normal((groups, m1))
        den = rng.standard_normal((groups, n))
        return x, u, num, den

    # --- random instances mirroring pkg/tests/conftest.py:random_instance --------
    run_case("f64_2x3x8_g2", *rnd((2, 3, 8), 2, dtype=np.float64), groups=2, block=2, with_oracle=True)
    run_case("f32_3x5x8_g4", *rnd((3, 5, 8), 4), groups=4, block=4, with_oracle=True)
    run_case("f32_2x4x16_g2", *rnd((2, 4, 16), 2), groups=2, block=4, with_oracle=True)
    run_case("tail_f64_3x3x8_g2", *rnd((3, 3, 8), 2, dtype=np.float64), groups=2, block=4,
             with_oracle=True, note="B*N=9 with S=4 (pkg/tests/test_backward.py:117-126)")
    run_case("tail_f32_7x13x64_g8", *rnd((7, 13, 64), 8), groups=8, block=16,
             note="91 rows, ragged last block")
    run_case("f32_4x16x32_g4_workers", *rnd((4, 16, 32), 4), groups=4, block=8,
             note="pkg/tests/test_backward.py:128-138 shape")
    run_case("f32_8x16x64_g8_determinism", *rnd((8, 16, 64), 8), groups=8, block=16,
             note="pkg/tests/test_acceptance.py:232-252 shape")
    # --- degrees other than (5, 4) -------------------------------------------------
    run_case("deg32_f32_4x2x8_g2", *rnd((4, 2, 8), 2, m1=4, n=2), groups=2, block=2, with_oracle=True)
    run_case("deg50_f32_3x4x16_g4", *rnd((3, 4, 16), 4, m1=6, n=0), groups=4, block=3, with_oracle=True)
    run_case("deg00_f64_2x2x4_g1", *rnd((2, 2, 4), 1, m1=1, n=0, dtype=np.float64), groups=1, block=1,
             with_oracle=True)
    run_case("deg11_f32_2x3x6_g3", *rnd((2, 3, 6), 3, m1=2, n=1), groups=3, block=2, with_oracle=True)
    run_case("deg75_f32_2x8x16_g2", *rnd((2, 8, 16), 2, m1=8, n=5), groups=2, block=4,
             note="degrees above (5,4) exercise the generic-degree kernels")
    # --- odd group widths (scalar / non-vector paths) ------------------------------
    run_case("dg3_f32_5x7x12_g4", *rnd((5, 7, 12), 4), groups=4, block=8)
    run_case("dg5_f64_3x5x10_g2", *rnd((3, 5, 10), 2, dtype=np.float64), groups=2, block=4)
    run_case("dg12_f32_4x9x48_g4", *rnd((4, 9, 48), 4), groups=4, block=8,
             note="d_g=12: float4-aligned, not 8-aligned (bf16 scalar path)")
    # --- structured inputs ---------------------------------------------------------
    x = rng.standard_normal((2, 3, 8)).astype(np.float32)
    x.reshape(-1)[::5] = 0.0
    x.reshape(-1)[1::7] = -0.0
    num = np.zeros((2, 6)); num[:, 1] = 1.0
    run_case("identity_zeros_f32_2x3x8_g2", x, rng.standard_normal((2, 3, 8)).astype(np.float32),
             num, np.zeros((2, 4)), groups=2, block=2, with_oracle=True,
             note="identity params: A(x)=0, sign(0)=0 path; exact +/-0 inputs")
    x = rng.standard_normal((3, 4, 16)).astype(np.float32)
    x.reshape(-1)[::3] = 0.0
    x.reshape(-1)[1::11] = -0.0
    run_case("zeros_f32_3x4x16_g4", x, rng.standard_normal((3, 4, 16)).astype(np.float32),
             rng.standard_normal((4, 6)), rng.standard_normal((4, 4)), groups=4, block=4)
    u0 = np.zeros((2, 3, 8), dtype=np.float32)
    run_case("zero_upstream_f32", rng.standard_normal((2, 3, 8)).astype(np.float32), u0,
             rng.standard_normal((2, 6)), rng.standard_normal((2, 4)), groups=2, block=2)
    run_case("large_mag_f32_4x4x16_g2",
             rng.uniform(-1e3, 1e3, (4, 4, 16)).astype(np.float32),
             rng.standard_normal((4, 4, 16)).astype(np.float32),
             rng.uniform(-1e3, 1e3, (2, 6)), rng.uniform(-1e3, 1e3, (2, 4)), groups=2, block=4,
             note="pkg/tests/test_rational.py:56-69 magnitudes")
    run_case("routing_1x1x4_g2", np.array([[[1.0, 2.0, 3.0, 4.0]]]),
             np.ones((1, 1, 4)), np.array([[0, 1.0, 0, 0, 0, 0], [5.0, 0, 0, 0, 0, 0]]),
             np.zeros((2, 4)), groups=2, block=1, note="pkg/tests/test_rational.py:140-147")
    run_case("single_element_x3", np.array([[[3.0]]]), np.array([[[1.0]]]),
             np.array([[0, 1.0, 0, 0, 0, 0]]), np.zeros((1, 4)), groups=1, block=256,
             note="pkg/tests/test_backward.py:32-42")
    run_case("overflow_f32_4x4x1", np.full((4, 4, 1), 1.0e30, dtype=np.float32),
             np.ones((4, 4, 1), dtype=np.float32), np.array([[0, 1.0, 0, 0, 0, 0]]),
             np.zeros((1, 0)), groups=1, block=256, note="pkg/tests/test_backward.py:59-65")
    # --- presets (pkg/src/grkan/presets/*.coeffs) -------------------------------
    for target in ("identity", "swish", "gelu"):
        fit = load_builtin_preset(target)
        manifest["presets"][target] = {"numerator": [float(v) for v in fit.numerator],
                                       "denominator": [float(v) for v in fit.denominator],
                                       "fit_error": float(fit.fit_error)}
        num = np.tile(fit.numerator, (8, 1))
        den = np.tile(fit.denominator, (8, 1))
        xs = rng.standard_normal((4, 8, 64)).astype(np.float32) * 2.0
        run_case("preset_%s_f32_4x8x64_g8" % target, xs,
                 rng.standard_normal((4, 8, 64)).astype(np.float32), num, den, groups=8, block=8)
    # --- rounding-experiment pass (verification.py:384-389, SMALL_SHAPE seed 11) ---
    prng = np.random.default_rng([11, 0])
    xr = prng.standard_normal((16, 8, 32)).astype(np.float32)
    ur = prng.standard_normal((16, 8, 32)).astype(np.float32)
    run_case("rounding_small_seed11", xr, ur, prng.standard_normal((4, 6)),
             prng.standard_normal((4, 4)), groups=4, block=1,
             note="rounding_experiment SMALL_SHAPE pass 0, block=ceil(128/1024)")
    # --- KAT-T (config 0): inputs regenerated from the seed, outputs hashed ---------
    xk, uk, nk, dk = kat_t_inputs(0)
    run_case("katt_seed0_f32_8x197x192_g8", xk, uk, nk, dk, groups=8, block=256,
             store_inputs=False, store_outputs=False,
             note="run_bench seed 0, KAT-T shape; x/u regenerated by kat_t_inputs(0)")
    manifest["cases"]["katt_seed0_f32_8x197x192_g8"]["sha_x"] = sha(xk)
    manifest["cases"]["katt_seed0_f32_8x197x192_g8"]["sha_u"] = sha(uk)

    # --- scalar known-answer tests (eval_rational / elementwise_grads) --------------
    def scalar(x, u, a, b, tag):
        y = g.eval_rational(x, a, b)
        eg = g.elementwise_grads(x, u, a, b)
        manifest["scalars"].append({"tag": tag, "x": x, "u": u, "a": list(map(float, a)),
                                    "b": list(map(float, b)), "y": y, "d_x": eg.d_x,
                                    "d_a": [float(v) for v in eg.d_a],
                                    "d_b": [float(v) for v in eg.d_b]})

    scalar(2.0, 1.0, [1.0, 0, 0, 0, 0, 0], [0.0, 0, 0, 0], "constant numerator")
    scalar(3.0, 1.0, [0.0, 1, 0, 0, 0, 0], [0.0, 0, 0, 0], "identity")
    scalar(1.0, 1.0, [1.0, 1.0], [1.0], "hand case (1+1)/(1+|1|)")
    scalar(2.0, 1.0, [1.0, 2.0], [], "empty denominator")
    scalar(0.0, 1.0, list(rng.standard_normal(6)), list(rng.standard_normal(4)), "x=0")
    scalar(2.0, 0.0, list(rng.standard_normal(6)), list(rng.standard_normal(4)), "zero upstream")
    for k in range(40):
        scalar(float(rng.uniform(-5, 5)), float(rng.standard_normal()),
               list(rng.standard_normal(6)), list(rng.standard_normal(4)), "random %d" % k)

    # --- GRKB tensor dumps written by the reference (cli.py:104-129) ------------------
    from grkan.cli import write_tensor_dump
    for case, key, fname in (("f32_2x4x16_g2", "dx", "dx_f32_2x4x16.grkb"),
                             ("f64_2x3x8_g2", "x", "x_f64_2x3x8.grkb")):
        write_tensor_dump(os.path.join(HERE, fname), g.ActivationTensor(arrays["%s/%s" % (case, key)]))
        manifest.setdefault("grkb", {})[fname] = {"case": case, "key": key}

    np.savez_compressed(os.path.join(HERE, "grkan_golden.npz"), **arrays)
    with open(os.path.join(HERE, "grkan_golden.json"), "w") as fh:
        json.dump(manifest, fh, indent=1, sort_keys=True)
    print("wrote %d arrays, %d cases, %d scalar KATs" % (len(arrays), len(manifest["cases"]),
                                                         len(manifest["scalars"])))


if __name__ == "__main__":
    main()
