"""Seeded synthetic inputs shared by the tests and the oracle side (no pPCA arithmetic here)."""
from . import philox, generate, configs  # noqa: F401
