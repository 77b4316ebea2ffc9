"""B200-native pre-screening hot path of arXiv 1707.05647 (reference: ``starscreen``).

Drop-in for ``starscreen.screen()`` and its configuration / feature-set
surface.  The per-pixel, per-scale work runs in hand-written sm_100a CUDA
kernels behind a C ABI (include/starscreen_b200.h, libstarscreen_b200.so);
there is no CPU fallback.
"""

from .config import (
    MIN_PATCH_SIDE,
    MIN_RING_HALF_SIZE,
    Quantizer,
    ScreeningConfig,
    default_star_radius,
    ladder_sizes,
    patch_center_margins,
    quantize,
    ring_plan,
    round_half_up,
)
from .featureset import FeatureSet, RingBand, RingFeatureVector, build_feature_set
from .image import as_gray, std_dev
from .second_stage import MatchResult, match_candidates
from .pgm import PgmError, load_pgm, save_pgm, save_screen_outputs, screen_stats_payload, write_json_atomic
from .screening import (
    CandidateList,
    FlatTemplateError,
    PruneStats,
    ScreeningResult,
    SizeMasks,
    prune_stats,
    screen,
    screen_batch,
)

__all__ = [
    "MIN_PATCH_SIDE",
    "MIN_RING_HALF_SIZE",
    "Quantizer",
    "ScreeningConfig",
    "default_star_radius",
    "ladder_sizes",
    "patch_center_margins",
    "quantize",
    "ring_plan",
    "round_half_up",
    "FeatureSet",
    "RingBand",
    "RingFeatureVector",
    "build_feature_set",
    "as_gray",
    "std_dev",
    "PgmError",
    "load_pgm",
    "save_pgm",
    "save_screen_outputs",
    "screen_stats_payload",
    "write_json_atomic",
    "CandidateList",
    "FlatTemplateError",
    "PruneStats",
    "ScreeningResult",
    "SizeMasks",
    "prune_stats",
    "screen",
    "screen_batch",
    "MatchResult",
    "match_candidates",
]
