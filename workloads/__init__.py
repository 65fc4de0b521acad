"""Seeded synthetic inputs for the five BASELINE.json configurations.

This package holds input recipes only (point clouds, fields and the RFD
parameters of each config).  It contains none of the method's arithmetic and
is the one module both the CUDA path's tests/bench and the oracle consume.
"""

from .configs import CONFIGS, barycenter_inputs, make_config  # noqa: F401
