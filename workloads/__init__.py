"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

Holds none of the Krylov method's arithmetic (see rng.py / models.py)."""
from . import rng, models, configs  # noqa: F401
