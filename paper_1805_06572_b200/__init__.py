"""B200-native FCA / FastFCA EM (arXiv 1805.06572), drop-in for the hot path
of the reference package ``fastfca`` 0.1.0.

Two-source multichannel separation with full-rank spatial covariances:
``fastfca_run`` (joint-diagonalisation EM) and ``fca_run`` (frame-wise EM)
run entirely on the GPU through hand-written sm_100a CUDA kernels in
``lib/libfastfca_b200.so`` (C ABI: ``include/fastfca_b200.h``). Names,
signatures, layouts, return types and exceptions follow the reference
(``pkg/src/fastfca/__init__.py:10-77``) for everything on the EM path and
the STFT front / back end (``stft_analyze`` / ``stft_synthesize``, also on
the GPU); ``separate`` chains analysis -> init -> EM -> synthesis in HBM.
``init_from_masks`` (the direction-clustering initial model) runs on the
GPU as well, and so is the SDR metric (``sdr`` / ``sdr_pairing``) and the
benchmark sweep's compute (``benchmark_sweep``). The simulator, WAV I/O and
CLI are out of scope.
"""

from .conventional import e_step, fca_run, log_likelihood, m_step
from .errors import (BackendUnavailableError, ConfigurationError, DefinitenessError,
                     FastFcaError, MetricError, NonHermitianError, PipelineError, SingularMatrixError,
                     SingularMixtureError)
from .fast import (fast_e_step, fast_m_step_S, fast_m_step_v, fastfca_run, propagate_pencil,
                   transform_observations)
from .benchmark import benchmark_sweep
from .initializers import init_from_masks, init_from_masks_batch, init_random, init_random_batch
from .metrics import measure_rtf, sdr, sdr_pairing, sdr_pairing_device, sdr_pairs_device
from .pencil import PencilDecomposition, gevd_hpd, hermitian_eig, solve_hermitian_system
from .pipeline import separate, separate_device
from .sharding import fastfca_run_sharded, fca_run_sharded
from .stft import (sqrt_hann, stft_analyze, stft_analyze_device, stft_synthesize,
                   stft_synthesize_device)
from .types import (AudioBuffer, OpCounts, PosteriorMoments, SeparationResult, SpatialModel,
                    SpectrogramTensor)

__version__ = "0.1.0"

__all__ = [
    "AudioBuffer",
    "BackendUnavailableError",
    "ConfigurationError",
    "DefinitenessError",
    "FastFcaError",
    "NonHermitianError",
    "OpCounts",
    "PipelineError",
    "PencilDecomposition",
    "PosteriorMoments",
    "SeparationResult",
    "SingularMatrixError",
    "SingularMixtureError",
    "SpatialModel",
    "SpectrogramTensor",
    "e_step",
    "fast_e_step",
    "fast_m_step_S",
    "fast_m_step_v",
    "fastfca_run",
    "fca_run",
    "gevd_hpd",
    "hermitian_eig",
    "fastfca_run_sharded",
    "fca_run_sharded",
    "benchmark_sweep",
    "init_from_masks",
    "measure_rtf",
    "sdr",
    "sdr_pairing",
    "sdr_pairing_device",
    "sdr_pairs_device",
    "MetricError",
    "init_from_masks_batch",
    "init_random",
    "init_random_batch",
    "log_likelihood",
    "m_step",
    "propagate_pencil",
    "separate",
    "separate_device",
    "solve_hermitian_system",
    "sqrt_hann",
    "stft_analyze",
    "stft_analyze_device",
    "stft_synthesize",
    "stft_synthesize_device",
    "transform_observations",
]
