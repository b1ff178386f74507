"""paper_2404_17101_b200 -- B200-native FAST-BCC (PASGAL, arXiv 2404.17101).

Drop-in for the reference package's biconnectivity entry point
(pasgal.oracles.bcc_hopcroft_tarjan, oracles.py:119-201) built from hand-written sm_100a
CUDA kernels behind a C-ABI (include/pasgal_bcc.h).  See DESIGN.md.
"""

from .results import BccLabels, canonical_checksum, canonical_edge_partition, canonical_relabel, min_eid_to_partition
from .graph import (CONFIGS, DeviceGraph, Graph, csr_from_keys, gen_grid, gen_knn, gen_rmat, make_config,
                    symmetrize_edges)
from .bcc import (DeviceBcc, HostBuffers, canonical_checksum_device, canonicalize_device, connected_components, connected_components_device,
                  same_partition_device)
from .bcc import articulation_bytes_device, bcc, bcc_device, release_workspace, unpack_articulation, validate_device, validate_workspace_bytes, workspace_bytes

from .io import GraphFormatError, load_adj, load_bin, load_graph, save_adj, save_bin
from .pipeline import BccPipeline
from .bfs import UNREACHED, DistanceArray, GraphStats, VgcConfig, bfs, bfs_parallel, eccentricities, estimate_diameter

__all__ = [
    "GraphFormatError", "load_adj", "load_bin", "load_graph", "save_adj", "save_bin",
    "BccPipeline", "UNREACHED", "DistanceArray", "GraphStats", "VgcConfig", "bfs", "bfs_parallel", "eccentricities",
    "estimate_diameter",
    "BccLabels", "canonical_checksum", "canonical_edge_partition", "canonical_relabel", "min_eid_to_partition",
    "CONFIGS", "DeviceGraph", "Graph", "csr_from_keys", "gen_grid", "gen_knn", "gen_rmat", "make_config",
    "symmetrize_edges", "DeviceBcc", "HostBuffers", "connected_components", "connected_components_device", "canonical_checksum_device", "canonicalize_device", "same_partition_device", "articulation_bytes_device", "bcc", "bcc_device", "release_workspace", "unpack_articulation",
    "validate_device", "validate_workspace_bytes", "workspace_bytes",
]

__version__ = "0.1.0"
