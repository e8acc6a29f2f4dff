"""paper_2305_04966_b200 — a B200-native (sm_100a) implementation of the
packed-sample volume-rendering hot path of NerfAcc (arXiv 2305.04966).

The product is ``libnacc.so`` behind the C ABI in ``include/nacc.h``; this
package is its thin PyTorch binding (``api``) named after Algorithm 1
(P:15-50).  ``harness`` binds the bench's synthetic-field library.
"""
from .api import (  # noqa: F401
    GridSpec,
    MarchParams,
    OccupancyGrid,
    PackedSamples,
    accumulate_along_rays,
    filter_early_stop,
    importance_sample,
    occgrid_ray_bounds,
    max_merge,
    pdf_loss,
    launch_count,
    neg_log_eps,
    owner_slab,
    prepare_bits,
    render_weights,
    render_weights_alpha,
    render_fwd,
    render_bwd,
    rendering,
    sampling_occgrid,
    MAP_IDENTITY,
    MAP_LINDISP,
)
from ._lib import NaccError  # noqa: F401
