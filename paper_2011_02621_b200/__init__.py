"""B200-native amplitude evaluation for tensor-network-state circuit simulation
(arXiv 2011.02621), a drop-in for the ``tnsim`` reference package's
amplitude-evaluation path.

The public names mirror ``tnsim`` (circuit builder, gate absorption, path
search, overlap network, slicing, amplitudes); the contraction path runs on
sm_100a through ``libtnc.so`` (include/tnc.h).
"""

from .circuit import (Circuit, CircuitFormatError, CircuitGraph, Gate, SingleQubitGate, SplitGate,
                      cz_matrix, edge_key, fsim_matrix, fuse_single_qubit_gates, gate_split,
                      generate_lattice, generate_rqc, iswap_matrix, parse_circuit, pattern_rqc,
                      serialize_circuit, split_gate_matrix, square_patterns, sycamore53_graph,
                      sycamore_patterns)
from .network import (AmplitudeBatch, AmplitudeEngine, AmplitudeStats, CutPlan, CutPlanError,
                      TensorNetwork, build_overlap_network, compute_amplitude, compute_amplitudes,
                      contract_along_path, plan_cuts, slice_network)
from .pathfind import (NetworkShape, PathSearchError, connectivity, exhaustive_path_oracle,
                       find_optimal_path, neighbours, score_increment, treewidth_bound)
from .tensor import Tensor, TensorError, contract_pair, contraction_cost, svd_factorize
from .tns import TNSState, apply_gate, compress_edge, evolve, init_state, two_sided_evolve

__version__ = "0.1.0"
