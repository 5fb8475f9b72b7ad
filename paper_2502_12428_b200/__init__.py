"""B200-native batched quasi-F-split heights of quartic K3 surfaces (drop-in for qfsplit's hot path)."""
from .errors import DomainError, EngineUnavailableError, InternalInvariantError, ParseError, QfsplitError  # noqa: F401

__version__ = "0.1.0"
