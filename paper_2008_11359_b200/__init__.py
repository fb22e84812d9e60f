"""paper_2008_11359_b200 -- B200-native (sm_100a) gSpMM / gSDDMM / edge softmax,
the data-parallel hot path of FeatGraph (SC20, arXiv 2008.11359).

The product is libfg.so (C ABI, include/fg.h); this package is its thin
binding (fg.py) plus the in-tree build (build.py) and the dst-row sharding
helpers (shard.py).
"""
from .fg import (FGError, Graph, Comm, comm_unique_id, edge_softmax, edge_softmax_backward, gat_attention, lib,  # noqa: F401
                 sddmm, sddmm_backward, spmm, spmm_backward, FG_OK, FG_EINVAL, FG_ESHAPE, FG_EUNSUPPORTED,
                 FG_EGRAPH, FG_ECUDA, FG_ENOMEM, FG_ENCCL)
