"""B200-native RNG hot path of arXiv 2109.01329 (drop-in for portarng's
engine / distribution / kernel-plugin surface).

Importing the package loads libprng_b200.so (hand-written sm_100a CUDA
kernels behind a C ABI, include/prng_b200.h).  There is no CPU fallback: if
the library is missing the import fails.
"""

from ._kernels import IMPL as kernel_impl
from .distributions import (
    Gaussian,
    Lognormal,
    RandomBlock,
    Uniform,
    UniformBits,
    fill_gaussian,
    fill_lognormal,
    fill_uniform,
    fill_uniform_unit,
    gaussian_from_words,
    generate,
    range_transform,
    word_to_unit,
    words_consumed,
    words_to_unit,
)
from .engine import (
    EngineKind,
    Mrg32k3a,
    Mrg32k3aState,
    Philox4x32x10,
    PhiloxState,
    generate_words,
    mrg_unit,
    next_word,
    philox_block,
    seed_engine,
    skip_ahead,
    stream_position,
)
from .errors import Error, InvalidParameter, InvalidRange, UnsupportedEngine

__version__ = "0.1.0"

__all__ = [
    "EngineKind",
    "Error",
    "Gaussian",
    "InvalidParameter",
    "InvalidRange",
    "Lognormal",
    "Mrg32k3a",
    "Mrg32k3aState",
    "Philox4x32x10",
    "PhiloxState",
    "RandomBlock",
    "Uniform",
    "UniformBits",
    "UnsupportedEngine",
    "fill_gaussian",
    "fill_lognormal",
    "fill_uniform",
    "fill_uniform_unit",
    "gaussian_from_words",
    "generate",
    "generate_words",
    "kernel_impl",
    "mrg_unit",
    "next_word",
    "philox_block",
    "range_transform",
    "seed_engine",
    "skip_ahead",
    "stream_position",
    "word_to_unit",
    "words_consumed",
    "words_to_unit",
]
