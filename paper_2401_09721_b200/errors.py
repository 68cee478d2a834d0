"""Exception classes with the reference's names and ValueError ancestry.

Each maps 1:1 to a status code returned by the C ABI (include/fgbd_b200.h):
FGBD_E_CLOUD -> CloudError (cloud.py:13), FGBD_E_GRAPH -> GraphError
(graph.py:20), FGBD_E_NOISE -> NoiseEstimationError (noise.py:26),
FGBD_E_FILTER -> FilterError (filtering.py:25).  AllPointsExcludedError
(filtering.py:29) is raised only by the stand-alone `fslr_mask`; `denoise`
downgrades it to a warning exactly as the reference does.
"""


class CloudError(ValueError):
    """Invalid point cloud data or incompatible cloud pair."""


class GraphError(ValueError):
    """Invalid graph construction input or degenerate graph."""


class NoiseEstimationError(ValueError):
    """Patch construction or estimation cannot proceed."""


class FilterError(ValueError):
    """Filtering or selection cannot proceed."""


class AllPointsExcludedError(FilterError):
    """Every point was masked out; fall back to unmasked selection."""


class DeviceError(RuntimeError):
    """CUDA / NCCL failure inside the B200 library (no reference analogue)."""
