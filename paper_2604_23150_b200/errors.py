"""Exception hierarchy mirroring the reference's moeplace::Error classes
(/root/reference/proj/core/include/moeplace/errors.hpp:11-66); the C ABI's
status codes map 1:1 onto them (include/moeplace_b200.h, mpb_status)."""


class Error(RuntimeError):
    """moeplace::Error — base class of all library errors."""


class ParseError(Error):
    def __init__(self, line: int, what: str):
        super().__init__(f"line {line}: {what}")
        self.line = line


class ValidationError(Error):
    pass


class ConfigError(Error):
    pass


class EmptySelectionError(Error):
    pass


class UndefinedCorrelationError(Error):
    pass


class InfeasibleError(Error):
    pass


class LookupError_(Error):
    """moeplace::LookupError (trailing underscore: Python's LookupError is a builtin)."""


class CudaError(Error):
    """CUDA runtime failure inside the library (no reference analogue)."""


_BY_STATUS = {1: Error, 3: ValidationError, 4: ConfigError, 5: EmptySelectionError,
              6: UndefinedCorrelationError, 7: InfeasibleError, 8: LookupError_, 9: CudaError}


def raise_for_status(status: int, what: str) -> None:
    if status == 2:
        raise ParseError(0, what)
    raise _BY_STATUS.get(status, Error)(what)
