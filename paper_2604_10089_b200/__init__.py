"""paper_2604_10089_b200 -- B200-native LCP-MVP / Stokes-mobility hot path of arXiv 2604.10089.

The product is libbpqn.so (C ABI, include/bpqn.h; CUDA sources in csrc/).  This
package only marshals arguments to it (``_bpqn``).  It never imports ``oracle/``.
"""
from ._bpqn import (BpqnError, Geometry, contacts, default_disc_opts, default_gmres_opts,  # noqa: F401
                    default_solve_opts, dvi_step, geometry_init, geometry_shard, geometry_shard_nccl, geometry_update, gmres_recycle_reset, janus_slip, layer_apply, lcp_b, lcp_matrix_dense, lcp_mvp, lib,
                    mobility_apply, nccl_unique_id, profile_get, profile_reset, set_contacts, solve_lcp, solve_lcp_dense)
