"""Off-line ROM data model (mirror of reference rom.py:319-356 SubdomainModel).

The batched sm_100a build pipeline lives in ``romgpu.py`` / ``csrc/sfw_rom.cu``;
``build_subdomain_model`` keeps the reference signature (rom.py:359-364).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import NumericalError


@dataclass
class SubdomainModel:
    """Everything the online stage needs for one subdomain (rom.py:319-356).

    The chain stacks have shape (layers, 6m, 6m); ``basis`` is the node-space
    image V Q of the reduction basis (optional: only source / receiver
    subdomains need it, as in sim.load_models, sim.py:359-398).  ``tdiag`` /
    ``toff`` keep the block-Lanczos blocks (A_j, B_j), the best-conditioned
    parity targets.
    """

    alpha: tuple
    lo: tuple
    shape: tuple
    spacing: tuple
    modes_per_face: int
    layers: int
    shift: float
    neighbors: dict
    face_indices: tuple
    gammas: np.ndarray
    gamma_hats: np.ndarray
    scales: np.ndarray
    basis: np.ndarray | None
    c: np.ndarray
    mu: np.ndarray
    deflated: bool = False
    truncated: bool = False
    tdiag: np.ndarray | None = None
    toff: np.ndarray | None = None

    @property
    def width(self) -> int:
        return 6 * self.modes_per_face

    def face_slice(self, face: int) -> slice:
        m = self.modes_per_face
        return slice(face * m, (face + 1) * m)

    @property
    def state_size(self) -> int:
        return self.layers * self.width


def require_basis(model) -> np.ndarray:
    if getattr(model, "basis", None) is None:
        raise NumericalError("model was loaded without its node-space basis")
    return model.basis
