"""Exception types of the hot path, same names and meaning as the reference
(pkg/src/portarng/errors.py:4-17)."""


class Error(Exception):
    """Base class for all errors of this package (portarng.errors.Error)."""


class UnsupportedEngine(Error):
    """Operation is not available for the requested engine."""


class InvalidRange(Error):
    """Range bounds are reversed, equal or non-finite."""


class InvalidParameter(Error):
    """Distribution or simulation parameter out of domain."""
