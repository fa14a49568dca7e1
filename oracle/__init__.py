"""CPU oracle for the seethrough EM hot path -- TEST INFRASTRUCTURE ONLY.

This package is a plain numpy restatement of the reference algorithm
(`/root/reference/pkg/src/seethrough/{sampling,features,geometry,solver,refocus,prior}.py`).
Every function cites the reference file:line it follows.

Who may import it: `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` leg -- and there only as the checker or
the timed CPU baseline, never as the thing measured or shipped.  The product
package `paper_2003_11076_b200` never imports it and fails loudly when its
CUDA library is missing.

Pinning: the oracle is checked bit-for-bit against golden vectors produced by
running the reference itself in the build container
(`tests/golden/make_golden.py`, fixtures `tests/golden/*.npz`), and, when
`/root/reference` is present, directly against the reference on fresh seeds
(`tests/test_oracle.py`).
"""

from .em import (  # noqa: F401
    DESC_LEN, DESC_MARGIN, RING, VARIANCE_CEILING, STATUS_VALID,
    STATUS_LOW_TEXTURE, STATUS_NO_STATIC_EVIDENCE, PROV_FALLBACK, PROV_COPIED,
    PROV_REFOCUSED, OracleParams, warp, bilinear, gray_of, sobel_of,
    descriptors_of, log_prior, e_step, e_step_scores, mask_order,
    OracleSolver, synthesize, median_filter, mu_raster, numpy_sum_order,
)
