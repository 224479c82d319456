"""Error taxonomy of the engine.

Mirrors the three exception classes of the reference package
(reference: pkg/src/flatlog/errors.py:1-29) so callers can catch the same
names; the CLI-style exit-code mapping is program=1, input=2, internal=3.
"""


class DatalogError(Exception):
    """Root of every error raised by this package."""


class ProgramError(DatalogError):
    """The Datalog source is malformed: syntax, arity, safety, strata, splits.

    When a source position is known the message is prefixed "line:col: ",
    the same convention as the reference's ProgramError.
    """

    def __init__(self, message, line=None, col=None):
        self.line = line
        self.col = col
        if line is not None:
            where = str(line) if col is None else f"{line}:{col}"
            message = f"{where}: {message}"
        super().__init__(message)


class InputError(DatalogError):
    """Bad facts or inputs (file problems, arity, symbol-space exhaustion)."""


class InternalError(DatalogError):
    """An engine invariant failed (count/materialize divergence, corrupt
    storage, device errors). Never the user's fault."""


class DeviceUnavailable(InternalError):
    """The sm_100a library or a CUDA device is missing. The engine has no
    CPU fallback, so this is raised instead of silently degrading."""


# drop-in alias for code written against the reference package
FlatlogError = DatalogError
