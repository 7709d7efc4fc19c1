"""B200-native TAGC compressed gradient exchange (arXiv 2504.05638).

The product is libtagc_b200.so: sm_100a CUDA kernels for threshold select,
split + encode (packed index + count sketch), NCCL exchange and the peeling
decoder, behind the C-ABI in include/tagc_b200.h. This package is the Python
host mirror of the reference API used by tests and bench.py.
"""
from .api import *  # noqa: F401,F403
from .api import Context, CompressionConfig, LayerSpec, LayerSegment, ShardSpec, PeelStats  # noqa: F401
from .specs import gpt2_specs, llama3_8b_specs  # noqa: F401

__version__ = "0.1.0"
