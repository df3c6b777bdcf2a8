"""B200-native noisy density-matrix gate engine: the data-parallel hot path of TANQ-Sim
(arXiv 2404.13184).  The product is the C-ABI library libtanq.so (include/tanq.h); this
package is its thin Python binding (paper_2404_13184_b200.tanq)."""
from .tanq import Simulator, TanqError, CReadout, QasmCircuit, Device, nccl_unique_id, lib  # noqa: F401
