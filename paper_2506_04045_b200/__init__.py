"""B200-native GPA/FISTA solver for similarity-based fuzzy clustering (arXiv 2506.04045).

Drop-in for the reference's hot path (/root/reference/proj/include/fuzzyclust:
share_matrix, fused_column_pass, gpa_step(_fused), project_simplex, run_gpa,
run_fista, solve).  Compute runs in hand-written sm_100a kernels behind the C
ABI in include/fuzzyclust_cuda.h (csrc/), loaded from lib/libfuzzyclust_cuda.so.
"""
from .errors import DeviceError, InvalidInput, IoError
from .similarity import SparseSimilarity
from . import capi
from .api import (
    ColumnPass, InitKind, InitStrategy, Method, SolverConfig, SolverResult, SolverTrace, TerminationReason,
    TraceRecord, default_context, default_step_size, feasibility_error, fista_t_next, fused_column_pass,
    generate_citation, generate_sbm, gpa_step, gpa_step_fused, init_membership, kReductionBlock, kVersion,
    loss_decomposed, project_simplex, read_membership_csv, resolve_step_size, run_fista, run_gpa,
    set_default_context, share_frob_sq, share_matrix, solve, splitmix64_doubles, splitmix64_stream, to_string,
    validate_membership, write_membership_csv, write_trace_csv, write_membership_binary, read_membership_binary,
    write_similarity_binary, read_similarity_binary, from_triplets, build_similarity,
    cross_share, hessian_vector_product, quadratic_form, frob_inner,
    Graph, ParsedGraph, LoadedGraph, parse_edge_list, largest_connected_component_nodes, two_core_nodes,
    induced_subgraph, largest_connected_component, prune_degree_one, load_pipeline, write_edge_list,
    SecondOrderConfig, RefinementStatus, RefinementVerdict, RefinementReport, full_gradient, projection_residual,
    is_critical, is_interior, refine,
)
