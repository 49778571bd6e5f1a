"""paper_2510_16028_b200 -- B200-native (sm_100a) hot path of NAO (arXiv 2510.16028).

Per operator of a traced FP32 forward: a sound IEEE-754 bound, the bound /
percentile-threshold check, and the Merkle commitment of the traced tensor,
behind the reference fpverify API (bounds / calibration / dispute /
commitments).  Kernels live in the in-tree C-ABI library libnao_b200.so
(include/nao_b200.h); there is no CPU fallback.
"""

from .bounds import (BoundTensor, FpModel, co_execute, gamma, gamma_tilde, layernorm_bound_parts,
                     matmul_bound, op_bound, softmax_bound, softmax_bound_parts)
from .calibration import (PERCENTILE_GRID, OpThresholds, ThresholdSet, percentile,
                          percentile_profile)
from .commitments import (MerkleProof, MerkleTree, build_tree, canon_tensor, commit_tensors,
                          leaf_digest, prove, tensor_root, trace_root, verify)
from .dispute import check_node, leaf_check, observed_p_max, p_max, screen, select_offending
from .engine import NATIVE, DeviceProfile, ExecutionError, default_profiles
from .graph import Graph, OpNode, Slice, build_graph, frontiers, make_node, partition
from .tensor import Rng, Tensor, tensor_new

__version__ = "0.1.0"
