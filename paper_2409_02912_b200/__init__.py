"""B200-native (sm_100a) neural-receiver (NRX) forward pass.

Drop-in for ``nrxsim.nrx.nrx_forward`` of the reference package
(/root/reference/pkg/src/nrxsim/nrx.py:345-385): a received resource grid
plus pilot/MCS configuration in, per-UE LLRs and a refined channel estimate
out, computed by hand-written CUDA kernels in ``libnrx_b200.so`` behind the
C ABI of ``include/nrx_b200.h``.
"""

from .config import (McsEntry, NrxConfig, PilotBook, SlotConfig, checkpoint_load, checkpoint_save,
                     default_mcs_table, expected_shapes, extended_mcs_table, generate_pilots,
                     init_weights)

__all__ = ["McsEntry", "NrxConfig", "PilotBook", "SlotConfig", "checkpoint_load", "checkpoint_save",
           "default_mcs_table", "expected_shapes", "extended_mcs_table", "generate_pilots",
           "init_weights", "nrx_forward", "NrxEngine"]


def __getattr__(name):
    # the GPU entry points import torch lazily
    if name == "nrx_forward":
        from .nrx import nrx_forward
        return nrx_forward
    if name == "NrxEngine":
        from .engine import NrxEngine
        return NrxEngine
    raise AttributeError(name)
