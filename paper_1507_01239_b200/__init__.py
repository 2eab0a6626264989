"""paper_1507_01239_b200 — B200-native model-averaging DNN trainer
(arXiv:1507.01239 path of the reference ``parnn`` library).

The compute path is ``libparnn_b200.so`` (hand-written sm_100a CUDA: tcgen05
GEMMs with fused epilogues, NG-SGD, RBM CD-1, NCCL averaging) behind the C ABI
in ``include/parnn_b200.h``. ``parnn`` mirrors the reference API on top of it.
"""
from ._lib import LIB_PATH, ParnnError, lib  # noqa: F401
from . import parnn  # noqa: F401
