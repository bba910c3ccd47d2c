"""paper_1404_0774_b200 — a B200-native fractal (PIFS) image encoder/decoder.

Drop-in for the encode/decode path of the reference `fic` codec
(proj/python/fic/__init__.py): the same public names, backed by sm_100a CUDA kernels
through the C-ABI in include/fic_b200.h (libfic_b200.so, built in-tree).
"""
from .codec import (
    CodecError,
    CodecParams,
    EncodedImage,
    collage_error,
    decode,
    decode_step,
    decode_traced,
    decode_timing,
    decoded_error_bound,
    encode,
    encode_batch,
    encode_device,
    encode_batch_device,
    encode_range,
    encode_rows,
    encode_with_stats,
    kernel_launch_count,
    last_survivors,
    matcher_timing,
    psnr,
    rmse,
    scan_timing,
    set_device,
    set_matcher_timing,
    validate_geometry,
)
from .pgm import load_pgm, write_pgm

__all__ = [
    "CodecError",
    "CodecParams",
    "EncodedImage",
    "collage_error",
    "decode",
    "decoded_error_bound",
    "encode",
    "load_pgm",
    "psnr",
    "rmse",
    "validate_geometry",
    "write_pgm",
    # extensions
    "decode_step",
    "decode_timing",
    "decode_traced",
    "encode_batch",
    "encode_device",
    "encode_batch_device",
    "encode_range",
    "encode_rows",
    "encode_with_stats",
    "kernel_launch_count",
    "last_survivors",
    "matcher_timing",
    "scan_timing",
    "set_device",
    "set_matcher_timing",
]
