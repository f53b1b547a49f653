/*
 * C restatement of the GR-KAN reference algorithm -- TEST INFRASTRUCTURE ONLY.
 *
 * The checker for the CUDA path at sizes where the NumPy oracle is slow (full
 * KAT-B: 155M elements).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it; the product library never links it.
 *
 * Built by oracle/Makefile with -ffp-contract=off and SSE math (no x87, no
 * fast-math), so every *, +, / rounds separately in the tensor precision and
 * the results reproduce the NumPy reference bit for bit (
 * pinned against tests/golden by tests/test_oracle_golden.py).
 *
 *   rational_values        pkg/src/grkan/rational.py:218-224
 *   gradient_terms         pkg/src/grkan/rational.py:227-278
 *   forward_tensor         pkg/src/grkan/rational.py:325-345
 *   backward_naive         pkg/src/grkan/backward.py:187-246
 *   backward_blocked       pkg/src/grkan/backward.py:275-372
 *   reference_coeff_grads  pkg/src/grkan/verification.py:318-341
 */
#include <math.h>
#include <stdint.h>

#define MAXC 32

/* double first: its helpers also serve the "true fp64" fold of the float instance */
#define REAL double
#define SUF dbl
#include "grkan_oracle_body.h"
#undef REAL
#undef SUF

#define REAL float
#define SUF f
#include "grkan_oracle_body.h"
#undef REAL
#undef SUF
