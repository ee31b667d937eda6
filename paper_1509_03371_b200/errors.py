"""The reference's exception taxonomy (common.hpp:9-31).

The C ABI maps these to status codes (SPEC 2, IO 3, NUMERIC 4, SIZE 6); ``_lib.check`` raises
them again with the reference's message text.
"""


class Error(RuntimeError):
    """pixelseg::Error"""


class SpecError(Error):
    """pixelseg::SpecError: bad network/solver specs, inconsistent geometry, invalid arguments."""


class SizeError(SpecError):
    """pixelseg::SizeError: shape/size violations detected while wiring or running a net."""


class IoError(Error):
    """pixelseg::IoError"""


class NumericError(Error):
    """pixelseg::NumericError"""
