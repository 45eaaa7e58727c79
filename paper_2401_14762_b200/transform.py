"""Dictionaries for the GPU solvers: an orthonormal basis plus measurement masks.

Mirrors the reference's dictionary layer (`hypercs/transform.py`) for the hot
path: `Dictionary` (`transform.py:220-264`), `build_dictionary`
(`:267-281`), `SelectionMask` / `build_selection_mask` (`:100-136`),
`measure` (`:168-173`) and `lipschitz_constant` (`:176-217`).

Differences, all B200-driven and documented in DESIGN.md:

* the basis is real and orthonormal (the BASELINE configs use the orthonormal
  DCT-II, `DctBasis`); the reference's complex DFT is not supported on the
  device path;
* a dictionary may carry one mask per pixel (`Dictionary.per_pixel`), which is
  what BASELINE's measurement model needs; the reference's single shared mask
  is the special case;
* the GPU never materialises A_p = Psi[mask_p, :]: kernels read Psi (L2
  resident) and the uint8 masks.  `Dictionary.from_matrix` therefore accepts
  any matrix with orthonormal rows (completing it to an orthonormal basis),
  and rejects others with ValueError.
"""

from dataclasses import dataclass, field

import numpy as np

from . import synth

ORTHO_TOL = 1e-10


@dataclass
class DctBasis:
    """Orthonormal real basis Psi (n x n), f = Psi @ c (cf. DftBasis, transform.py:19-30)."""

    n: int
    matrix: np.ndarray

    def __post_init__(self):
        if self.n < 1:
            raise ValueError("basis size must be >= 1")
        if self.matrix.shape != (self.n, self.n):
            raise ValueError("basis matrix shape mismatch")


def build_dct_basis(n):
    """Orthonormal DCT-II synthesis basis of size n (BASELINE's Psi)."""
    if n < 1:
        raise ValueError("basis size must be >= 1")
    return DctBasis(n=n, matrix=synth.dct_basis(n))


@dataclass
class SelectionMask:
    """Sorted subset of spectral sample indexes (transform.py:100-119)."""

    n: int
    indices: np.ndarray
    seed: int

    def __post_init__(self):
        self.indices = np.asarray(self.indices, dtype=np.intp)
        if self.indices.ndim != 1 or self.indices.size == 0:
            raise ValueError("mask needs at least one index")
        if self.indices.min() < 0 or self.indices.max() >= self.n:
            raise ValueError("mask index out of range")
        if np.any(np.diff(self.indices) <= 0):
            raise ValueError("mask indices must be strictly increasing")

    @property
    def m(self):
        return int(self.indices.size)


def build_selection_mask(n, ratio, seed):
    """Seeded selection of round-half-up(ratio * n) indexes (transform.py:122-136)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    if not 0.0 < ratio <= 1.0:
        raise ValueError("ratio must be in (0, 1]")
    m = int(np.floor(ratio * n + 0.5))
    if m < 1:
        raise ValueError("ratio keeps no samples")
    rng = np.random.default_rng(seed)
    return SelectionMask(n=n, indices=np.sort(rng.choice(n, size=m, replace=False)), seed=seed)


def measure(f, mask):
    """y = f[mask.indices] (transform.py:168-173), real-valued here."""
    f = np.asarray(f, dtype=np.float64)
    if f.shape != (mask.n,):
        raise ValueError("spectrum length does not match the mask")
    return f[mask.indices]


def _check_orthonormal(basis):
    n = basis.shape[0]
    err = np.abs(basis.T @ basis - np.eye(n)).max()
    if err > ORTHO_TOL:
        raise ValueError(f"basis is not orthonormal (max |Psi^T Psi - I| = {err:.2e})")


def _as_real(matrix):
    matrix = np.asarray(matrix)
    if np.iscomplexobj(matrix):
        if np.any(matrix.imag != 0):
            raise ValueError("the GPU backend needs a real dictionary")
        matrix = matrix.real
    return np.ascontiguousarray(matrix, dtype=np.float64)


def _complete_basis(rows):
    """Orthonormal n x n basis whose first m rows are `rows` (orthonormal)."""
    m, n = rows.shape
    if m == n:
        return rows.copy()
    # orthogonal complement of the row space
    q, _ = np.linalg.qr(np.concatenate([rows.T, np.eye(n)], axis=1))
    comp = q[:, m:n].T
    comp -= (comp @ rows.T) @ rows
    q2, _ = np.linalg.qr(comp.T)
    return np.concatenate([rows, q2.T[: n - m]], axis=0)


@dataclass(frozen=True)
class AdmmFactor:
    """(A_p^T A_p + alpha I)^-1 = Psi^T diag(1 / (d_p + alpha)) Psi."""

    alpha: float
    dictionary: object = field(repr=False)

    def diagonal(self, p=0):
        d = np.zeros(self.dictionary.n)
        m = self.dictionary.masks if self.dictionary.shared else self.dictionary.masks[p]
        d[m.astype(np.intp)] = 1.0
        return 1.0 / (d + self.alpha)

    def solve(self, b, p=0):
        psi = self.dictionary.basis
        return psi.T @ (self.diagonal(p) * (psi @ b))


@dataclass
class Dictionary:
    """A_p = basis[mask_p, :] for every pixel p.

    ``masks`` is either one sorted index vector (the reference's shared mask,
    `.matrix` available) or a (P, m) uint8 array of per-pixel masks.
    ``lipschitz`` is computed on the GPU on first access (power iteration of
    transform.py:176-217; = 1 up to rounding for orthonormal bases).
    """

    basis: np.ndarray
    masks: np.ndarray
    mask: SelectionMask | None = None
    _lipschitz: object = None
    _admm_factors: dict = field(default_factory=dict, repr=False)
    _device: dict = field(default_factory=dict, repr=False)

    def __post_init__(self):
        self.basis = _as_real(self.basis)
        n = self.basis.shape[0]
        if self.basis.shape != (n, n):
            raise ValueError("basis must be square")
        if n > 256:
            raise ValueError("the GPU backend supports n <= 256 bands")
        _check_orthonormal(self.basis)
        masks = np.asarray(self.masks)
        if masks.ndim not in (1, 2) or masks.shape[-1] < 1:
            raise ValueError("masks must be (m,) or (P, m)")
        if masks.min() < 0 or masks.max() >= n:
            raise ValueError("mask index out of range")
        if masks.shape[-1] > 1 and np.any(np.diff(masks.astype(np.int64), axis=-1) <= 0):
            raise ValueError("mask indices must be strictly increasing")
        self.masks = masks.astype(np.uint8)

    # ---- reference-compatible surface (transform.py:220-264) ---------------
    @property
    def shared(self):
        return self.masks.ndim == 1

    @property
    def m(self):
        return int(self.masks.shape[-1])

    @property
    def n(self):
        return int(self.basis.shape[0])

    @property
    def n_pixels(self):
        return None if self.shared else int(self.masks.shape[0])

    @property
    def matrix(self):
        if not self.shared:
            raise ValueError("a per-pixel dictionary has no single matrix; use matrix_of(p)")
        return self.basis[self.masks.astype(np.intp), :]

    def matrix_of(self, p):
        m = self.masks if self.shared else self.masks[p]
        return self.basis[m.astype(np.intp), :]

    @property
    def lipschitz(self):
        """Power-iteration constant(s) of A (GPU); a float for a shared mask."""
        if self._lipschitz is None:
            from .kernels import lipschitz_batch
            masks = self.masks[None, :] if self.shared else self.masks
            vals = lipschitz_batch(self.basis, masks)
            self._lipschitz = float(vals[0]) if self.shared else vals
        return self._lipschitz

    def admm_factor(self, alpha):
        """The ADMM system (A^T A + alpha I) in factored form, cached per alpha.

        For orthonormal Psi, A^T A + alpha I = Psi^T diag(d + alpha) Psi with d
        the mask indicator, so the factor is the diagonal 1 / (d + alpha): the
        GPU solves with two basis products instead of a triangular pair
        (transform.py:253-264 caches a Cholesky factor instead).
        """
        if alpha <= 0:
            raise ValueError("alpha must be > 0")
        f = self._admm_factors.get(alpha)
        if f is None:
            f = AdmmFactor(alpha=alpha, dictionary=self)
            self._admm_factors[alpha] = f
        return f

    # ---- constructors --------------------------------------------------------
    @classmethod
    def from_matrix(cls, matrix):
        """Wrap a dense matrix with orthonormal rows (transform.py:245-251).

        The rows are completed to an orthonormal basis Psi and the mask selects
        them, so A = Psi[mask, :] exactly."""
        rows = _as_real(matrix)
        if rows.ndim != 2:
            raise ValueError("dictionary matrix must be 2-D")
        m, n = rows.shape
        if m > n or np.abs(rows @ rows.T - np.eye(m)).max() > ORTHO_TOL:
            raise ValueError("the GPU backend needs a dictionary with orthonormal rows "
                             "(a row selection of an orthonormal basis)")
        return cls(basis=_complete_basis(rows), masks=np.arange(m))

    @classmethod
    def per_pixel(cls, basis, masks):
        """One mask per pixel: A_p = basis[masks[p], :] (BASELINE's measurement model)."""
        b = basis.matrix if isinstance(basis, DctBasis) else basis
        masks = np.asarray(masks)
        if masks.ndim == 3:
            masks = masks.reshape(-1, masks.shape[-1])
        return cls(basis=b, masks=masks)

    # ---- device residency ----------------------------------------------------
    def pinned_masks(self):
        """Per-pixel masks as a pinned host tensor (pinned once, cached): the
        host pipeline of recover_cube copies them to the device every call
        with asynchronous DMA instead of a staged pageable copy."""
        import torch
        hit = self._device.get("pinned")
        if hit is None:
            hit = torch.from_numpy(np.ascontiguousarray(self.masks)).pin_memory()
            self._device["pinned"] = hit
        return hit

    def device_arrays(self, device, n_pixels):
        """(basis, masks) as CUDA tensors; masks broadcast to n_pixels rows."""
        import torch
        key = (str(device), n_pixels)
        hit = self._device.get(key)
        if hit is None:
            basis = torch.as_tensor(self.basis, device=device)
            if self.shared:
                masks = torch.as_tensor(self.masks, device=device).unsqueeze(0).expand(n_pixels, -1).contiguous()
            else:
                if self.masks.shape[0] != n_pixels:
                    raise ValueError("per-pixel masks do not match the number of pixels")
                masks = torch.as_tensor(self.masks, device=device)
            hit = (basis, masks)
            # one device copy at a time (the pinned host copy stays)
            self._device = {k: v for k, v in self._device.items() if k == "pinned"}
            self._device[key] = hit
        return hit


def build_dictionary(basis, mask, alpha=None):
    """Dictionary of the basis rows kept by the mask (transform.py:267-281)."""
    b = basis.matrix if isinstance(basis, DctBasis) else np.asarray(basis)
    if mask.n != b.shape[0]:
        raise ValueError("mask and basis sizes differ")
    d = Dictionary(basis=b, masks=mask.indices, mask=mask)
    if alpha is not None:
        d.admm_factor(alpha)
    return d


def lipschitz_constant(matrix):
    """Largest eigenvalue of A^T A (transform.py:176-217) for a matrix with
    orthonormal rows, computed by the GPU power-iteration kernel."""
    return Dictionary.from_matrix(matrix).lipschitz
