"""fp64 CPU oracle — TEST INFRASTRUCTURE ONLY (see rf_oracle.py header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package.  It shares no code with paper_2110_01899_b200/.
"""
from .rf_oracle import *  # noqa: F401,F403
from .rf_oracle import (ACTS, sigma, dsigma, d2sigma, hermite_rule, gauss_expect, moments,  # noqa: F401
                        moments_trapezoid, tau_hat, sigma_features, gram, gram_entries, gram_schmidt,
                        eq1_terms, eq1, phi_eq1, phi_eq2, phi_exact_pair, phi_pivot_asymmetry)
