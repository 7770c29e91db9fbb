"""Exception hierarchy mirroring the reference's errors.hpp:10-59.

The C ABI (include/dashsvd_b200.h) returns integer status codes; the host
layer re-raises them as these types so callers see the same contract as the
reference library (e.g. the CLI's exit-code mapping, tools/dashsvd.cpp:404-422).
"""


class Error(RuntimeError):
    """Base class for every error raised by this library (errors.hpp:10-13)."""


class ParseError(Error):
    def __init__(self, line: int, what: str):
        super().__init__(f"parse error at line {line}: {what}")
        self.line = line


class UnsupportedFormat(Error):
    pass


class ShapeError(Error):
    """Dimension mismatch or a shape precondition violated (errors.hpp:27-30)."""


class ConfigError(Error):
    """Invalid solver configuration (errors.hpp:32-35)."""


class RankDeficient(Error):
    """eigSVD rank floor hit; ``index`` is the 0-based singular value (errors.hpp:37-43)."""

    def __init__(self, index: int, what: str):
        super().__init__(f"{what} (index {index})")
        self.index = index


class NumericalError(Error):
    """Non-convergence or non-finite intermediates (errors.hpp:45-49)."""


class DegenerateReference(Error):
    pass


class HypothesisError(Error):
    pass


class DeviceError(Error):
    """CUDA / NCCL / out-of-memory failure inside the B200 path (no reference analogue;
    the reference maps these to its base Error)."""


class UnsupportedOnDevice(Error):
    """A configuration the B200 path does not implement (e.g. l > 512, QR with l > 160, the basic
    algorithm on a row-sharded matrix)."""
