"""ORACLE (test infrastructure only) — see oracle/krylov.py header.

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  Independent of the CUDA library.
"""
from .krylov import (arnoldi, evolve, find_step, integrand, omega, one_norm,  # noqa: F401
                     small_eig, spmv, tanh_sinh)
