"""Record the reference's access-model predictions and instrumented counts.

Imports the reference package (``grkan``, /root/reference/pkg/src) in the build
container only; the committed ``access_golden.json`` travels instead.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_access_golden.py

Per case: ``predict_accesses_naive`` (pkg/src/grkan/access.py:89),
``predict_accesses_blocked`` (:97, or the TailNotCoveredError it raises),
``predicted_total_for_plan`` (:119) and, for small shapes, the counts
``instrumented_backward`` (:129) observes while running each strategy.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

# (batch, seq, feature, groups, block_size, m1, n, instrument)
CASES = [
    (1, 9, 8, 2, 4, 6, 4, True),     # tail block (test_backward.py:117-126 geometry)
    (2, 8, 16, 4, 4, 6, 4, True),    # exact tiling
    (1, 5, 12, 3, 2, 3, 2, True),    # other degrees, tail
    (8, 197, 192, 8, 256, 6, 4, False),    # KAT-T
    (128, 197, 1536, 8, 256, 6, 4, False),  # KAT-S hidden
    (256, 197, 3072, 8, 256, 6, 4, False),  # KAT-B hidden
    (256, 197, 3072, 8, 197, 6, 4, False),  # exact tiling at KAT-B
]


def main() -> None:
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF_SRC)
    from grkan import access, backward, rational
    from grkan.errors import TailNotCoveredError

    out = []
    for batch, seq, feature, groups, bs, m1, n, instrument in CASES:
        mc = m1 + n
        case = {"batch": batch, "seq": seq, "feature": feature, "groups": groups, "block_size": bs,
                "m1": m1, "n": n,
                "naive": access.predict_accesses_naive(batch, seq, feature, mc)}
        try:
            case["blocked"] = access.predict_accesses_blocked(batch, seq, feature, bs, feature // groups, mc)
        except TailNotCoveredError:
            case["blocked"] = None
        layout = rational.GroupLayout(feature, groups)
        for strategy in ("blocked", "naive"):
            plan = getattr(backward.ExecutionPlan, strategy)(batch, seq, layout, bs)
            case["plan_" + strategy] = access.predicted_total_for_plan(batch, seq, feature, plan, mc)
            if instrument:
                rng = np.random.default_rng(batch * 1000 + seq * 10 + feature)
                x = rational.ActivationTensor(rng.standard_normal((batch, seq, feature)).astype(np.float32))
                u = rational.ActivationTensor(rng.standard_normal((batch, seq, feature)).astype(np.float32))
                params = rational.GroupRationalParams(rng.standard_normal((groups, m1)),
                                                      rng.standard_normal((groups, n)))
                _, rep = access.instrumented_backward(x, u, params, plan)
                case["instrumented_" + strategy] = rep.to_dict()
        out.append(case)
    with open(os.path.join(HERE, "access_golden.json"), "w") as f:
        json.dump({"source": "grkan.access (pkg/src/grkan/access.py)", "cases": out}, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main()
