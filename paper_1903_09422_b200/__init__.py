"""B200-native KADABRA adaptive-sampling betweenness engine (arXiv:1903.09422 hot path).

    from paper_1903_09422_b200 import adsamp
    parsed = adsamp.parse_edge_list_file("graph.edges")
    cfg = adsamp.EngineConfig(variant=adsamp.Variant.indexed, samples_per_frame=1, base_seed=42)
    res = adsamp.kadabra.estimate_bc(parsed.graph, 0.01, 0.1, cfg)

All compute goes through libadsb.so (include/adsb.h): hand-written sm_100a
kernels for the sampler, the ordered cutoff and the epoch check, NCCL for
multi-GPU runs. Importing this package does not load the library; the first
call does, and fails loudly if it has not been built.
"""
from . import adsamp, kadabra  # noqa: F401
from ._lib import (AdsbError, CudaError, DomainError, InvalidArgument, LogicError,  # noqa: F401
                   NcclError, ParseError)

__all__ = ["adsamp", "kadabra", "AdsbError", "CudaError", "DomainError", "InvalidArgument", "LogicError",
           "NcclError", "ParseError"]
