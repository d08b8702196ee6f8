"""Exception hierarchy with the reference's names (src/errors.py:11-44).

The C-ABI returns status codes (include/sts_b200.h); ``raise_for_status``
maps them onto these classes so callers catch exactly what they caught with
the reference: 1 -> ConfigError (an InputError), 2 -> ContractViolation.
"""

from __future__ import annotations


class SpecSparseError(Exception):
    """Base class for all package errors (src/errors.py:11)."""


class InputError(SpecSparseError):
    """User-supplied input is invalid (src/errors.py:15; CLI exit 1)."""


class ContractViolation(SpecSparseError):
    """An internal precondition was violated (src/errors.py:19; CLI exit 2)."""


class CapacityError(InputError):
    """A sequence or cache would exceed its capacity (src/errors.py:23)."""


class ConfigError(InputError):
    """A configuration object is inconsistent or infeasible (src/errors.py:27)."""


class DeviceError(SpecSparseError):
    """A CUDA runtime failure inside the native library (status 3)."""


STS_OK, STS_ERR_INPUT, STS_ERR_CONTRACT, STS_ERR_CUDA = 0, 1, 2, 3


def raise_for_status(code: int, message: str) -> None:
    if code == STS_OK:
        return
    if code == STS_ERR_INPUT:
        raise ConfigError(message)
    if code == STS_ERR_CONTRACT:
        raise ContractViolation(message)
    raise DeviceError(message or f"native error {code}")
