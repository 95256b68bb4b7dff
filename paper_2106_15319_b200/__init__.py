"""B200-native serial-EMD (arXiv 2106.15319) hot path.

serialize -> sift (EMD / EEMD / CEEMDAN) -> noise-ensemble mean -> IMF store
-> deserialize, as hand-written sm_100a CUDA behind the reference's API
(see include/semd_b200.h for the C ABI and api.py for the Python mirror).
"""
from .api import (CapacityError, Context, EngineError, InsufficientExtrema, InvalidInput, ceemdan, concatenate,
                  concatenate_naive, context, deconcatenate, decompose, decompose_full, default_transition_length,
                  derive_seed, eemd, emd, envelope, extract_imf, find_extrema, noise_mode, parse_algorithm,
                  serial_decompose, serial_decompose_full, signal_std, slicewise_decompose, transition_weights,
                  white_noise)

__all__ = [
    "CapacityError", "Context", "EngineError", "InsufficientExtrema", "InvalidInput", "ceemdan", "concatenate",
    "concatenate_naive", "context", "deconcatenate", "decompose", "decompose_full", "default_transition_length",
    "derive_seed", "eemd", "emd", "envelope", "extract_imf", "find_extrema", "noise_mode", "parse_algorithm",
    "serial_decompose", "serial_decompose_full", "signal_std", "slicewise_decompose", "transition_weights",
    "white_noise",
]
