"""B200-native incircle RayCast, traversal and Monte-Carlo integration.

Drop-in for the hot path of the reference package ``voronray``
(pkg/src/voronray/__init__.py:3-32): the RayCast, full-diagram traversal and
MC volume/area entry points keep their names, arguments, return types and
exceptions, and run as hand-written sm_100a kernels behind a C-ABI library
(include/voronray_b200.h) loaded with ctypes.  There is no CPU fallback.
"""

from . import errors, rng
from .core import (TOL_VERTEX, TOL_DEGENERATE, HALFSPACE_SLACK, BoundaryRay, Mesh, NodeSet,
                   VertexRecord, build_node_set, edge_keys, nearest_neighbor, verify_vertex,
                   verify_vertices)
from .raycast import (RayQuery, RaycastBatch, RaycastStats, initial_heuristic, project_t,
                      raycast_batch, raycast_incircle, search_direction, vertex_directions_batch)
from .graph import (DESCENT_RETRIES, VerifyReport, brute_force_vertices, circumcenters, descent,
                    descent_batch, edge_set, set_sub_rounds, verify_mesh, voronoi_graph,
                    voronoi_local)
from .integrate_mc import (CellIntegrals, Integrand, MCResult, mc_areas_only, mc_cells,
                           mc_directions, mc_integrals_cells, mc_integrate_cell, mc_uniforms,
                           sample_unit_sphere, sphere_surface_area)
from . import integrands, io
from .integrate_hmc import (HMCResult, face_index, hmc_cell_integral, hmc_cells,
                            hmc_interface_integral, hmc_volume)

__version__ = "0.1.0"

__all__ = [
    "Mesh", "NodeSet", "VertexRecord", "BoundaryRay", "build_node_set", "nearest_neighbor",
    "verify_vertex", "verify_vertices", "TOL_VERTEX", "TOL_DEGENERATE", "HALFSPACE_SLACK",
    "edge_keys", "RayQuery", "RaycastStats", "RaycastBatch", "project_t", "initial_heuristic",
    "raycast_incircle", "raycast_batch", "search_direction", "vertex_directions_batch",
    "edge_set", "descent", "descent_batch", "voronoi_graph", "voronoi_local", "verify_mesh",
    "VerifyReport", "set_sub_rounds",
    "brute_force_vertices", "circumcenters", "DESCENT_RETRIES", "CellIntegrals", "Integrand",
    "MCResult", "sample_unit_sphere", "sphere_surface_area", "mc_areas_only", "mc_cells",
    "mc_directions", "mc_integrate_cell", "mc_integrals_cells", "mc_uniforms", "integrands",
    "errors", "rng", "io", "hmc_volume", "hmc_interface_integral", "hmc_cell_integral",
    "hmc_cells", "HMCResult", "face_index",
]
