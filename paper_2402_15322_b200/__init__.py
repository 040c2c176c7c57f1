"""B200-native entropic optimal transport on SE(2) (arXiv 2402.15322): the Sinkhorn /
convolutional Wasserstein-barycenter scaling loop as hand-written sm_100a CUDA behind the C ABI
in include/se2ot.h, with this thin Python binding on top (argument marshalling only).

    from paper_2402_15322_b200 import Kernel, se2_conv, se2_sinkhorn, se2_barycenter, ...
"""
from .api import (Kernel, make_porous_prox, make_prox, se2_bary_logmean, se2_bary_update, se2_barycenter, se2_conv,
                  se2_conv_update, se2_jko_step, se2_kernel_build, se2_launch_count, se2_marginal_error,
                  se2_scale_rows, se2_sinkhorn, se2_sum, se2_sum_rows, se2_transport_cost, se2_barycenter_precise,
                  se2_conv_precise)
from ._lib import SE2Error, LIB_PATH
from .lifting import (Cake, interpolate_images, se2_exp, se2_log, se2_lift_field, se2_lift_image, se2_project,
                      se2_project_signed, se2_reconstruct_field, se2_split_signed)

__all__ = ["Kernel", "make_porous_prox", "make_prox", "se2_bary_logmean", "se2_bary_update", "se2_barycenter", "se2_conv",
           "se2_conv_update", "se2_jko_step", "se2_kernel_build", "se2_launch_count", "se2_marginal_error",
           "se2_sinkhorn", "se2_sum", "se2_sum_rows", "se2_scale_rows", "se2_transport_cost", "se2_barycenter_precise",
           "se2_conv_precise", "SE2Error",
           "LIB_PATH", "Cake", "interpolate_images", "se2_exp", "se2_log", "se2_lift_field", "se2_lift_image", "se2_project",
           "se2_project_signed", "se2_reconstruct_field", "se2_split_signed"]
