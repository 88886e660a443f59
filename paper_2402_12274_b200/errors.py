"""Error taxonomy, kept code-for-code with the reference
(/root/reference/pkg/src/minimpi/errors.py:9-76) so callers dispatching on
``exc.code`` behave identically.  The integer values are the MPX_* status
codes of include/mpx.h.
"""


class MinimpiError(Exception):
    code = "ERR_OTHER"

    def __init__(self, msg="", *, status=None):
        super().__init__(msg or self.code)
        self.status = status


def _kind(name, code, doc):
    return type(name, (MinimpiError,), {"code": code, "__doc__": doc})


StateError = _kind("StateError", "ERR_STATE", "Object used outside its lifecycle.")
PendingError = _kind("PendingError", "ERR_PENDING", "Teardown with operations outstanding.")
ArgError = _kind("ArgError", "ERR_ARG", "Bad argument, bounds, wrong completion family.")
TransportError = _kind("TransportError", "ERR_TRANSPORT", "Transfer-path failure.")
SpawnError = _kind("SpawnError", "ERR_SPAWN", "Launcher could not start a participant.")
ExhaustedError = _kind("ExhaustedError", "ERR_EXHAUSTED", "Fixed-capacity pool is full.")
UnsupportedError = _kind("UnsupportedError", "ERR_UNSUPPORTED", "Recognised but unimplemented.")
TruncateError = _kind("TruncateError", "ERR_TRUNCATE", "Incoming data larger than the layout.")

# MPX_* integer status -> class (include/mpx.h)
_BY_INT = {1: ArgError, 2: StateError, 3: PendingError, 4: TruncateError,
           5: UnsupportedError, 6: ExhaustedError, 7: TransportError,
           8: MinimpiError}
_BY_CODE = {c.code: c for c in (MinimpiError, StateError, PendingError, ArgError,
                                TransportError, SpawnError, ExhaustedError,
                                UnsupportedError, TruncateError)}


def error_for_code(rc, msg=""):
    return _BY_INT.get(rc, MinimpiError)(msg)


def for_status(status):
    """Exception matching a completion status's error code."""
    cls = _BY_CODE.get(status.error, MinimpiError)
    return cls("operation completed with %s" % status.error, status=status)
