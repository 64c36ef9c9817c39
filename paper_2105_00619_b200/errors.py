"""Exception taxonomy mirroring include/optb/errors.hpp:9-42 of the reference.

The C ABI returns a status code plus the reference's what() text; the host
mirror re-raises the same class with the same message, so tests written
against the reference's messages (e.g. test_codec.cpp:128-134,
test_sampler.cpp:57-58) hold unchanged.
"""


class Error(RuntimeError):
    """optb::Error -- base of everything the library throws on purpose."""


class ShapeError(Error):
    """optb::ShapeError"""


class CapacityError(Error):
    """optb::CapacityError"""


class FormatError(Error):
    """optb::FormatError"""


class CudaError(Error):
    """CUDA runtime failure (no reference counterpart)."""


class ArgumentError(Error, ValueError):
    """Invalid argument to the C ABI itself (no reference counterpart)."""


_BY_CODE = {1: Error, 2: ShapeError, 3: CapacityError, 4: FormatError, 5: CudaError, 6: ArgumentError}


def raise_for(code: int, message: str):
    raise _BY_CODE.get(code, Error)(message)
