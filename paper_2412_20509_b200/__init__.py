"""B200-native aSGD hot path for penalized generalized matrix factorization
(arXiv 2412.20509), a drop-in for the reference package's ``fit_asgd`` path.

Host API (this package) mirrors gmfkit's names and error behaviour; the
compute runs in hand-written sm_100a CUDA kernels behind the C ABI declared in
include/gmf_asgd.h (libgmf_asgd.so, built in-tree).  There is no CPU
fallback: device entry points raise when the library or a GPU is missing.
"""
__version__ = "0.1.0"

from .exceptions import (ConfigError, DegenerateError, DivergenceError, DomainError,  # noqa: F401
                         GmfError, SingularSystemError)
from .families import (Bernoulli, FamilySpec, Gamma, Gaussian, Identity, Inverse,  # noqa: F401
                       InverseGaussian, InverseSquared, LinkSpec, Log, Logit, NegBinomial,
                       Poisson, canonical_link, ddot_d, dot_d, family, link)
from .gradients import GradientPair, Minibatch, full_gradients, minibatch_gradients  # noqa: F401
from .identify import check_constraints, project_constraints  # noqa: F401
from .model import (CovariateSet, FactorizationState, PenaltyConfig, ResponseMatrix,  # noqa: F401
                    parameter_count, penalty_value)
from .optim import (FitReport, SgdConfig, bias_correction, fit_asgd, impute_block,  # noqa: F401
                    learning_rate, linear_predictor, penalized_objective, smooth_update,
                    update_dispersion_stochastic, update_nb_shape_stochastic)
from .initialization import InitMethod, init_glm_svd, init_ols_svd  # noqa: F401
from .metrics import EvalResult, rel_deviance, rel_log_rmse  # noqa: F401
from .select import (RankSelectionReport, cv_rank_select, elbow_pick, holdout_mask,  # noqa: F401
                     information_criteria, residual_scores, scree_eigenvalues)
from .io import read_matrix_market, read_matrix_market_csr  # noqa: F401

__all__ = [name for name in dir() if not name.startswith("_")]
