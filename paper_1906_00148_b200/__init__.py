"""B200-native batched TFHE gate bootstrapping for SHE (arxiv 1906.00148).

The product is libshe.so (C-ABI in include/she.h; CUDA kernels for sm_100a in
csrc/); ``she`` is its thin ctypes binding.  See DESIGN.md.
"""
from . import she  # noqa: F401
from .she import (Context, she_decrypt_bits, she_encrypt_bits, she_gate_batch,  # noqa: F401
                  she_gate_batch_ops, she_gate_batch_ops_host, she_gate_level, she_keygen)
