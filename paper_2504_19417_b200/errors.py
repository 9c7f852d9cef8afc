"""Exception hierarchy of the drop-in (mirrors evflow/errors.py:4-29).

When the reference `evflow` package is importable, these classes also derive
from its exception types, so `except evflow.DimensionMismatchError` keeps
working for code switched over to this package.
"""

from __future__ import annotations


def _ref(name):
    try:  # optional: only for except-compatibility with the reference
        import evflow.errors as ref  # type: ignore
        return (getattr(ref, name),)
    except Exception:
        return ()


class EvflowError(*_ref("EvflowError"), Exception):
    """Base class for all errors of this package."""


class EventParseError(EvflowError, *_ref("EventParseError")):
    """A weight or event file could not be parsed."""


class GeometryError(EvflowError, *_ref("GeometryError")):
    """A coordinate does not fit the declared camera geometry."""


class DimensionMismatchError(EvflowError, *_ref("DimensionMismatchError")):
    """Embedding / weight / feature dimensions do not agree."""


class EmptyNeighborhoodError(EvflowError, *_ref("EmptyNeighborhoodError")):
    """A query event has no events in its spatiotemporal neighbourhood."""
