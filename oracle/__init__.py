"""Plain fp64 CPU oracle of the IPM hot path (arXiv 1912.09238).

TEST INFRASTRUCTURE ONLY — see ipm_oracle.h.  Never imported by the product
package ``paper_1912_09238_b200``.
"""
from .oracle import Oracle, build, clenshaw_curtis, farfield_ghost, gauss_legendre, multi_indices, num_basis, smolyak_cc  # noqa: F401
