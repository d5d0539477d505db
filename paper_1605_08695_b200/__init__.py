"""B200-native sharded-embedding + sampled-softmax training step (arXiv 1605.08695 §4.2, §6.4).

The hot path lives in ``libtfs.so`` (hand-written sm_100a CUDA behind the C ABI of
``include/tfs.h``); this package is its Python binding (``ops``) and the step driver
(``step``) that composes the calls -- Part -> route -> Gather -> route back -> Stitch ->
sampled softmax -> sort-reduce -> route -> ScatterAdd/SGD -- with torch used only for device
memory, streams and torch.distributed (NCCL) process groups.
"""
from . import _lib  # noqa: F401
from ._lib import (TFS_BF16, TFS_F32, TFS_REMOVE_ACCIDENTAL_HITS, TFS_SUBTRACT_LOG_Q,  # noqa
                   TfsError)

__all__ = ["ops", "step", "TfsError", "TFS_BF16", "TFS_F32", "TFS_SUBTRACT_LOG_Q",
           "TFS_REMOVE_ACCIDENTAL_HITS"]
