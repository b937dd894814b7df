"""B200-native DMD hot path (arXiv 2502.05339), drop-in for the reference
`flowdmd` fit/predict API on that path.

    from paper_2502_05339_b200 import SnapshotMatrix, exact_dmd, decode, encode, step_k
"""

from .dmd import (
    ControlOperator,
    LMConfig,
    ReducedModel,
    SnapshotMatrix,
    conjugate_pairs,
    dmdc_fit,
    exact_dmd,
    fit_control,
    optdmd,
    vandermonde,
)
from . import model_io
from .editing import EditSpec, apply_edit, band_energy, cluster_modes, omega
from .grid import GridSpec, MacField, ScalarField, coarse_grid, flatten, unflatten
from .serving import ModelServer, Session, shift_state
from . import solver
from .upres import UpresConfig, blend_fields, build_projector, constrained_project, guided_rollout, upres_step
from .errors import (
    BadMagicError,
    BadVersionError,
    ChecksumError,
    ConvergenceError,
    EigenvalueFloorError,
    FlowDmdError,
    FormatError,
    RolloutOverflowError,
    SizeMismatchError,
)
from .linalg import SvdResult, eig_small, lstsq, pinv, randomized_svd, truncated_svd
from .runtime import (
    ImaginaryResidueWarning,
    ModalBasis,
    ReducedState,
    continuous_coefficients,
    decode,
    decode_batch,
    encode,
    eval_continuous,
    inverse_step,
    kinetic_energy,
    reconstruct,
    rollout,
    step,
    step_forced,
    step_k,
)

__version__ = "0.1.0"
