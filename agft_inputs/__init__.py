"""Seeded input generators and named configs shared by the oracle and the CUDA path.

Holds constants and parameter tables only (no method arithmetic); see configs.py.
"""
from .configs import (BASE_SEED, named_config, tuner_params, with_overrides, frequencies,
                      tiny_config, live_inputs, ALPHA_GRID, TAU_E_GRID, K_H_GRID)

__all__ = ["BASE_SEED", "named_config", "tuner_params", "with_overrides", "frequencies",
           "tiny_config", "live_inputs", "ALPHA_GRID", "TAU_E_GRID", "K_H_GRID"]
