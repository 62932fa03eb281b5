"""B200-native (sm_100a) PDF inverse-scattering hot path.

Drop-in for the reference package's solver API on the per-iteration path
(physics loss forward + hand adjoint, corrective network, Adam), see DESIGN.md.
The setup modules (config, geometry, scenes, operators) import without a GPU;
the solver entry points load ``libpdfb200.so`` on first use and fail loudly
if it is missing.
"""
from .config import (C0, CcoParams, ConfigError, ImagingConfig, config_from_dict, config_hash, config_to_dict,
                     load_config, save_config)
from .geometry import AntennaArray, ComplexGrid, GridGeometry, build_array, build_grid, perturb_array
from .operators import (FieldSet, GeometryError, GreensOperators, NoConvergenceError, ScatteredData,
                        SingularSystemError,
                        SimulationResult, add_awgn, build_greens, incident_fields, plane_wave_fields,
                        simulate, solve_total_field, synthesize_scattered)
from .scenes import (Scene, SceneError, Shape, builtin_scene, ellipse, load_scene, rasterize, resolve_scene,
                     save_scene, scene_from_dict, scene_to_dict)

__version__ = "0.1.0"

_API = ("LossBreakdown", "LossContext", "PipelineState", "SpectralBasis", "NetworkParams", "AdamState",
        "ReconstructionResult", "BatchReconstructor", "pipeline_forward", "pipeline_backward", "grad_alpha",
        "loss_total", "init_network", "forward_net", "flatten_params", "unflatten_params", "grad_loss",
        "adam_step", "bp_initialize", "init_alpha", "recover_contrast", "apply_cco", "reconstruct",
        "relative_error", "count_components", "PoleError", "ZeroDataError", "PhysicsLoss", "truncate", "expand",
        "truncate_adjoint_scale", "apply_gd", "apply_gd_adjoint", "apply_gs_adjoint", "ContrastRecovery")


_CIE = ("chi_to_r", "r_to_chi", "default_eps_reg", "pixel_least_squares", "cie_state_residual")
_FILTERS = ("box_mean", "guided_filter")
_LOSSES = ("loss_data", "loss_state", "loss_bound", "loss_tv", "loss_bridge", "bound_chi_grad", "tv_chi_grad",
           "bridge_chi_grad", "regularizer_chi_grad")


def __getattr__(name):
    # the GPU API imports torch lazily so the setup modules stay light
    if name in _CIE:
        from . import cie
        return getattr(cie, name)
    if name in _FILTERS:
        from . import filters
        return getattr(filters, name)
    if name in _LOSSES:
        from . import losses
        return getattr(losses, name)
    if name == "CsiObjective":
        from .reconstruct import CsiObjective
        return CsiObjective
    if name in _API:
        from . import api
        return getattr(api, name)
    if name == "DeviceProblem":
        from .engine import DeviceProblem
        return DeviceProblem
    raise AttributeError(name)
