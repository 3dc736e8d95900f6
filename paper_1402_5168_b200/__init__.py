"""B200-native apply phase of the rational time-evolution operator
exp(tau L) u ~ sum_m b_m (tau L - alpha_m)^{-1} u  (Haut, Babb, Martinsson,
Wingate; PAPER.md).  The compute lives in librexp.so (include/rexp.h); this
package is the thin Python binding.
"""
from .api import Handle, apply, free, setup, step_finish, step_partial  # noqa: F401
