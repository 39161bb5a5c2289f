"""Former names of the native engine and predictor.  `engine.Engine` and
`predictor.Predictor` ARE libsppipe now (there is no other control plane);
these aliases keep older callers working."""
from __future__ import annotations

from .engine import _CLASS, Engine as NativeEngine  # noqa: F401
from .predictor import Predictor as NativePredictor  # noqa: F401
