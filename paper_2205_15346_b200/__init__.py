"""B200-native restarted-Krylov engine for v(t) = exp(-iHt) v (after TimeEvolver,
arXiv:2205.15346).  The product is libtimeevolver.so (include/te.h); ``te`` is its
ctypes binding."""
from . import te  # noqa: F401
