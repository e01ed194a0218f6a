"""B200-native (sm_100a) densification hot path of ImprovedGS+ (arXiv 2603.08661).

A drop-in for the densification path of the reference ``splitkit`` package
(``/root/reference/pkg/src/splitkit``): the edge-importance map, budgeted
split-candidate selection and Long-Axis-Split, with the reference's names,
arguments and exceptions.  Host code is Python; the arithmetic runs in
hand-written CUDA kernels in ``libigs_b200.so`` (C ABI: ``include/igs_b200.h``),
bound with ctypes.  There is no CPU fallback.
"""

from .core import Scene2, Scene3
from .densify_controller import (EVENT_CSV_HEADER, DensifyEvent, DensifyStats,
                                 accumulate_grads, accumulate_position_grads, densify_step,
                                 select_candidates)
from .edge_pipeline import (GradientField, blur_kernel_5x5, gaussian_blur_5x5,
                            importance_batch, importance_pipeline, median_normalize,
                            nms_thin, sample_scores, sobel_gradients, to_grayscale)
from .las_split import (BudgetError, SplitConstants, las_split_batch, las_split_batch_2d,
                        principal_axis)
from .scene_io import (BadMagicError, FormatError, SceneFormatError, SizeMismatchError,
                       UnsupportedVersionError, read_scene, scene_bytes, write_scene)
from .schedule import (DensifyConfig, ExpSchedule, default_schedules, is_densify_step,
                       is_warmup_step, lr_at)
from .splat2d import (RenderParams, TrainConfig, TrainResult, backward,
                      desk_scale_densify_config, loss_l2, psnr, render, ssim, train)
from .io_cli import read_image, write_image

__version__ = "0.1.0"
