"""B200-native S-fraction multiscale ROM wave solver (arXiv 1406.6923 path).

Drop-in for the reference ``sfwave`` hot path (pkg/src/sfwave/__init__.py:33-43):
the off-line per-subdomain ROM build and the on-line coupled leapfrog, both
executed by hand-written sm_100a CUDA in ``libsfw_b200.so`` (C ABI:
include/sfw_b200.h).  There is no CPU fallback: without the library or a CUDA
device every compute entry point raises ``DeviceError``.
"""

__version__ = "0.1.0"

from .errors import (ConfigError, DataError, DeviceError, InstabilityError, NumericalError,  # noqa: F401
                     ProtocolError, SfwaveError)
from .grid import (DomainPartition, DomainSpec, SubdomainOperator, assemble_global_operator,  # noqa: F401
                   assemble_subdomain_operator, build_partition, opposite_face)
from .fdtd import (FineGridOperator, LeapfrogRun, estimate_lambda_max, leapfrog_energy, run_leapfrog,  # noqa: F401
                   stability_limit)
from .io import TraceRecord, load_model, read_traces, save_model, write_traces  # noqa: F401
from .rom import (SubdomainModel, build_models, build_subdomain_model, project_state,  # noqa: F401
                  state_to_nodes)
from .stepper import (CoupledStepper, Probe, SourceTerm, cfl_estimate_coupled, make_probe,  # noqa: F401
                      project_source, resolve_dt, stable_step_coupled)

__all__ = [
    "ConfigError", "CoupledStepper", "DataError", "DeviceError", "DomainPartition", "DomainSpec",
    "FineGridOperator", "LeapfrogRun", "TraceRecord", "assemble_global_operator", "estimate_lambda_max",
    "leapfrog_energy", "load_model", "read_traces", "run_leapfrog", "save_model", "stability_limit",
    "write_traces",
    "InstabilityError", "NumericalError", "Probe", "ProtocolError", "SfwaveError", "SourceTerm",
    "SubdomainModel", "SubdomainOperator", "build_models", "build_subdomain_model", "assemble_subdomain_operator", "build_partition",
    "cfl_estimate_coupled", "make_probe", "opposite_face", "project_source", "project_state", "resolve_dt",
    "stable_step_coupled", "state_to_nodes",
    "__version__",
]
