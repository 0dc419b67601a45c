"""Seeded synthetic input generators (shared by the oracle tests, the GPU tests and bench.py).

This module holds NO arithmetic of the bilateral-filter method: it only draws images with the
shapes, value ranges and structure that BASELINE.json's five configs describe (ramp +
rectangles + noise; sinusoids + rectangles + noise). The paper's own images (Lena, Barbara,
Boat) are not available, so these stand in for them ("Inputs").
"""
from .generators import (CONFIGS, ramp_image, sinusoid_image, config_input, config_params,
                         ConfigSpec)

__all__ = ["CONFIGS", "ramp_image", "sinusoid_image", "config_input", "config_params", "ConfigSpec"]
