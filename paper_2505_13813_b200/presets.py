"""Built-in coefficient rows for the GR-KAN init modes.

Values are the fitted (m, n) = (5, 4) rows shipped with the reference
(pkg/src/grkan/presets/{identity,swish,gelu}.coeffs, parsed there by
load_coeff_preset, pkg/src/grkan/layer.py:226-247).  The paper initialises the
first rational of a KAT block to identity and the second to swish
(PAPER.md:470).  ``tests/test_host.py`` checks these numbers against the
golden manifest recorded from the reference.
"""

from __future__ import annotations

PRESETS = {
    "identity": {
        "numerator": (0.0, 1.0, 0.0, 0.0, 0.0, 0.0),
        "denominator": (0.0, 0.0, 0.0, 0.0),
        "fit_error": 0.0,
    },
    "swish": {
        "numerator": (3.2637916821290114e-07, 0.5000000000000003, 0.24999736015666932,
                      0.05326511838281725, 0.005802538653465898, 0.00027513311367496045),
        "denominator": (-5.027048134681183e-13, 0.10653023676588584, -4.9085854614779824e-14,
                        0.000550266227353655),
        "fit_error": 1.1841025586434295e-06,
    },
    "gelu": {
        "numerator": (-0.0004251030626581786, 0.5000000000043914, 0.4026986437032256,
                      0.07376487764405487, -0.01288387457622922, -0.003728354917937935),
        "denominator": (-5.92128467140623e-10, 0.14752975578371683, -1.3588916460591336e-10,
                        -0.007456709823817984),
        "fit_error": 0.0009213253182394077,
    },
}


def preset_row(name: str, degrees: tuple[int, int] = (5, 4)):
    """(numerator, denominator) tuples for an init mode; identity works at any degree."""
    m, n = degrees
    if name == "identity":
        if m < 1:
            raise ValueError("identity needs numerator degree >= 1")  # rational.py:118-119
        num = [0.0] * (m + 1)
        num[1] = 1.0
        return tuple(num), (0.0,) * n
    if name not in PRESETS:
        raise ValueError("unknown init %r (identity, swish, gelu)" % (name,))
    if (m, n) != (5, 4):
        raise ValueError("preset %r is fitted for degrees (5, 4), not %r" % (name, degrees))
    return PRESETS[name]["numerator"], PRESETS[name]["denominator"]
