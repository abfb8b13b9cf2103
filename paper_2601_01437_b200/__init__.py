"""B200-native IRL stochastic-reconfiguration hot path (arXiv 2601.01437).

Drop-in for the data-parallel core of the reference package ``irlnqs``:
``estimators`` (SampleBatch, estimate_energy, energy_gradient, heff_matvec,
qgt_matvec), ``krylov`` (lanczos, implicit_restart, irl_smallest),
``optimizer`` (bordered operator, IRL solve, update direction) and
``ansatz`` (RBM / shallow-MLP batched log-derivative rows).  The arithmetic
runs in the sm_100a C-ABI library ``libirlsr.so`` (include/irl_sr.h).
"""

__version__ = "0.1.0"

from . import _lib  # noqa: F401
