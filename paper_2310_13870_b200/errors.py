"""Error hierarchy mirroring proj/include/fsg/common.hpp:13-66.

Each class carries the reference's exit code: 2 config, 3 I/O, 4 numeric;
5 is this framework's device failure (no CUDA device, CUDA error, missing
extension).
"""


class Error(RuntimeError):
    exit_code = 1

    def __init__(self, msg: str = "", exit_code: int | None = None):
        super().__init__(msg)
        if exit_code is not None:
            self.exit_code = exit_code


class ConfigError(Error):
    exit_code = 2


class InvalidConfig(ConfigError):
    pass


class TooFewPoints(ConfigError):
    pass


class LengthMismatch(ConfigError):
    pass


class IoError(Error):
    exit_code = 3


class NumericError(Error):
    exit_code = 4


class DeviceError(Error):
    exit_code = 5


def error_for(code: int, msg: str) -> Error:
    if code == 2:
        if "n >= 2" in msg:
            return TooFewPoints(msg)
        return InvalidConfig(msg)
    if code == 3:
        return IoError(msg)
    if code == 4:
        return NumericError(msg)
    if code == 5:
        return DeviceError(msg)
    return Error(msg, code)
