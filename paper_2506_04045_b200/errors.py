"""Error convention of the reference API (common.hpp:11-20).

``IoError`` for unreadable input / parse failures, ``InvalidInput`` for shape,
config and feasibility failures and for non-finite projection input.  The C-ABI
returns 1 / 2 for these and 3 for a CUDA or NCCL failure (``DeviceError``).
"""


class IoError(RuntimeError):
    pass


class InvalidInput(RuntimeError):
    pass


class DeviceError(RuntimeError):
    pass


def raise_for(code: int, msg: str) -> None:
    if code == 0:
        return
    if code == 1:
        raise IoError(msg)
    if code == 2:
        raise InvalidInput(msg)
    raise DeviceError(msg)
