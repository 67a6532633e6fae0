"""Exception hierarchy mirroring the reference's
(/root/reference/proj/include/agentsim/common.hpp:25-130), mapped from the
C-ABI status codes of include/sutradhara_b200.h."""


class SimError(RuntimeError):
    pass


class ConfigError(ValueError):
    pass


class CacheError(SimError):
    pass


class CacheFull(CacheError):
    pass


class UnknownBlock(CacheError):
    pass


class ZeroRefRelease(CacheError):
    pass


class EngineError(SimError):
    pass


class StaleHandle(EngineError):
    pass


class InvalidState(EngineError):
    pass


class UnknownCall(EngineError):
    pass


class CudaError(RuntimeError):
    pass


class Unsupported(ValueError):
    pass


_BY_STATUS = {1: CacheFull, 2: UnknownBlock, 3: ZeroRefRelease, 4: CacheError, 5: ConfigError, 6: CudaError,
              7: ValueError, 8: Unsupported, 9: StaleHandle, 10: InvalidState, 11: UnknownCall}

STATUS_OF = {v: k for k, v in _BY_STATUS.items()}


def from_status(status: int, msg: str) -> Exception:
    return _BY_STATUS.get(status, RuntimeError)(msg)
