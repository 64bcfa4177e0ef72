"""paper_1805_11144_b200 — B200-native executor for the per-timestep step
loop of a merged Signal/Operator graph (the reference's EngineCore<T>)."""
from . import ir  # noqa: F401
