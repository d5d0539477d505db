"""B200-native sharded-embedding + sampled-softmax training step (arXiv 1605.08695 §4.2, §6.4).

The hot path lives in ``libtfs.so`` (hand-written sm_100a CUDA behind the C ABI of
``include/tfs.h``), including the native step runtime (tfs_comm / tfs_step_*) that composes
the calls -- sample -> Part -> route -> Gather -> route back -> Stitch -> sampled softmax ->
per-id gradient sums -> route -> ScatterAdd/SGD -- on its own streams, barriers and CUDA graph.
This package is its Python binding: ``ops`` (one function per entry point) and ``step`` (the
stepper and communicator), argument marshalling only; torch provides tensors over the library's
memory and torch.distributed the one-time exchange of the communicator's IPC handles.
"""
from . import _lib  # noqa: F401
from ._lib import (TFS_BF16, TFS_F32, TFS_REMOVE_ACCIDENTAL_HITS, TFS_SUBTRACT_LOG_Q,  # noqa
                   TfsError)

__all__ = ["ops", "step", "TfsError", "TFS_BF16", "TFS_F32", "TFS_SUBTRACT_LOG_Q",
           "TFS_REMOVE_ACCIDENTAL_HITS"]
