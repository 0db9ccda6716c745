"""SPEC-named exceptions of the ICCL path and the C result-code mapping.

Names follow the reference SPEC: the verbs errors
(SPEC.md:154), transport errors, monitor errors
(SPEC.md:326, 335), collectives, pipeline
and the cli ConfigError.  ``IcclError`` is the common base, as
``SimulationError`` is in the reference (engine.py:13-14).
"""
from __future__ import annotations


class IcclError(RuntimeError):
    code = -1

    def __init__(self, msg: str = "", code: int = None):
        super().__init__(msg)
        if code is not None:
            self.code = code


class InvalidArgument(IcclError, ValueError):
    code = 1


class CudaError(IcclError):
    code = 2


class SystemError_(IcclError):
    code = 3


class QpInErrorState(IcclError):
    code = 4


class UnregisteredRegion(IcclError):
    code = 5


class ZeroLengthMessage(IcclError, ValueError):
    code = 6


class ConnectionFailed(IcclError):
    code = 7


class UnknownWr(IcclError):
    code = 8


class TargetQpDead(IcclError):
    code = 9


class NonPositiveDuration(IcclError, ValueError):
    code = 10


class WindowNotFull(IcclError, ValueError):
    code = 11


class GroupTooSmall(IcclError, ValueError):
    code = 12


class NoSmAvailable(IcclError):
    code = 13


class InvalidConfig(IcclError, ValueError):
    code = 14


class ConfigError(IcclError, ValueError):
    code = 15


class SizeMismatch(IcclError, ValueError):
    code = 16


class IcclTimeout(IcclError, TimeoutError):
    code = 17


class InProgress(IcclError):
    code = 18


class Aborted(IcclError):
    code = 19


_BY_CODE = {cls.code: cls for cls in (
    InvalidArgument, CudaError, SystemError_, QpInErrorState, UnregisteredRegion, ZeroLengthMessage,
    ConnectionFailed, UnknownWr, TargetQpDead, NonPositiveDuration, WindowNotFull, GroupTooSmall,
    NoSmAvailable, InvalidConfig, ConfigError, SizeMismatch, IcclTimeout, InProgress, Aborted)}


def raise_for(code: int, where: str = "") -> None:
    """Raise the SPEC-named exception for a non-zero iccl_result_t."""
    if code == 0:
        return
    from ._lib import lib
    name = lib.iccl_get_error_string(code).decode()
    detail = (lib.iccl_get_last_error() or b"").decode()
    cls = _BY_CODE.get(code, IcclError)
    raise cls(f"{where}: {name}" + (f" ({detail})" if detail else ""), code)
