"""Drop-in host API of the reference solver, running on the B200 library.

Mirrors ``gdwd.solver`` / ``gdwd.subsolvers`` (reference
``pkg/src/gdwd/solver.py:44-602`` and ``subsolvers.py:32-55,283-364``): same
names, same dataclasses and defaults, same error behaviour.  Everything the
iteration touches runs in ``libgdwd_b200.so`` (include/gdwd_b200.h); this
module only validates inputs, moves the problem to the device once, and
assembles the returned records.  Scalar host helpers that the reference
computes once per problem (class weights, scaling, sigma rule for external
callers, backend selection) are plain Python here as well.
"""

from __future__ import annotations

import ctypes as C
import enum
import math
import threading
import time
import weakref
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _lib
from .model import FeatureMeta, ModelFile, identity_meta
from .sparse import SparseMatrixCSC, as_csc


# ---------------------------------------------------------------------------
# exceptions (reference solver.py:44, subsolvers.py:38, cholesky.py:12,
# lanczos.py:25)
# ---------------------------------------------------------------------------
class SingleClassError(ValueError):
    """Both classes must be present."""


class IndefiniteMatrixError(ArithmeticError):
    """The matrix has a non-positive-definite pivot."""


class DegenerateSchurError(ArithmeticError):
    """Schur-complement scalar is numerically zero or negative."""


class LanczosConvergenceError(RuntimeError):
    """Requested accuracy not reached."""


class SolverKind(enum.Enum):
    DIRECT = "direct"
    SMW2 = "smw2"
    ITERATIVE = "iterative"


def select_solver(n: int, d: int) -> SolverKind:
    """subsolvers.py:42-55: SMW2 if d > 5000 and 5n < d and n <= 2500;
    ITERATIVE if d > 5000; else DIRECT."""
    if n < 1 or d < 1:
        raise ValueError("n and d must be at least 1")
    if d > 5000 and 5 * n < d and n <= 2500:
        return SolverKind.SMW2
    if d > 5000:
        return SolverKind.ITERATIVE
    return SolverKind.DIRECT


class Backend(enum.Enum):
    AUTO = "auto"
    DIRECT = "direct"
    SMW2 = "smw2"
    ITERATIVE = "iterative"

    def resolve(self, n: int, d: int) -> SolverKind:
        if self is Backend.AUTO:
            return select_solver(n, d)
        return SolverKind(self.value)


@dataclass(frozen=True)
class ProblemData:
    """Scaled training problem (solver.py:60-95): ``z_tilde`` is d x n with
    column i equal to ``y_i x_i / z_scale``."""

    z_tilde: SparseMatrixCSC
    y: np.ndarray
    e: np.ndarray
    weights: np.ndarray
    C: float
    q: float
    z_scale: float

    def __post_init__(self):
        object.__setattr__(self, "y", np.asarray(self.y, dtype=np.float64))
        object.__setattr__(self, "e", np.asarray(self.e, dtype=np.float64))
        object.__setattr__(self, "weights", np.asarray(self.weights, dtype=np.float64))
        n = self.z_tilde.ncols
        if self.y.shape != (n,) or not np.all(np.isin(self.y, (-1.0, 1.0))):
            raise ValueError("labels must be a length-n vector over {-1,+1}")
        if self.e.shape != (n,) or np.any(self.e <= 0):
            raise ValueError("e must be positive of length n")
        if not np.isclose(self.e.max(), 1.0):
            raise ValueError("e must be normalized to max-norm 1")
        if self.weights.shape != (n,) or np.any(self.weights <= 0):
            raise ValueError("weights must be positive of length n")
        if not (self.C > 0 and self.q > 0 and self.z_scale > 0):
            raise ValueError("C, q and z_scale must be positive")

    @property
    def n(self) -> int:
        return self.z_tilde.ncols

    @property
    def d(self) -> int:
        return self.z_tilde.nrows


_GOLDEN = (1.0 + math.sqrt(5.0)) / 2.0


@dataclass(frozen=True)
class SolverConfig:
    """solver.py:101-124 (same fields, defaults and validation)."""

    q: float = 1.0
    max_iter: int = 2000
    steplength: float = 1.618
    tol_feas: float = 1e-5
    tol_cgap: float = math.sqrt(1e-5)
    tol_cap: float = 0.05
    sigma0: Optional[float] = None
    epsilon_c: Optional[float] = None
    backend: Backend = Backend.AUTO
    use_sgs: bool = True
    ell: int = 10
    mu: float = 1.0
    psqmr_switch_steps: int = 50
    seed: int = 0

    def __post_init__(self):
        if not 0.0 < self.steplength <= 1.618034:
            raise ValueError(f"steplength must lie in (0, {_GOLDEN:.6f})")
        if min(self.tol_feas, self.tol_cgap, self.tol_cap) <= 0:
            raise ValueError("tolerances must be positive")
        if self.q <= 0 or self.mu <= 0 or self.ell < 1 or self.max_iter < 1:
            raise ValueError("q, mu must be positive; ell, max_iter at least 1")


@dataclass
class SolverState:
    r: np.ndarray
    xi: np.ndarray
    alpha: np.ndarray
    w: np.ndarray
    u: np.ndarray
    rho: np.ndarray
    beta: float
    sigma: float
    iter: int
    eps_c: float


@dataclass(frozen=True)
class KKTResiduals:
    eta_c1: float
    eta_c2: float
    eta_c3: float
    eta_p1: float
    eta_p2: float
    eta_p3: float
    eta_d1: float
    eta_d2: float
    eta_gap: float
    obj_primal: float
    obj_dual: float

    @property
    def eta_p(self) -> float:
        return max(self.eta_p1, self.eta_p2, self.eta_p3)

    @property
    def eta_d(self) -> float:
        return max(self.eta_d1, self.eta_d2)

    @property
    def eta_c(self) -> float:
        return max(self.eta_c1, self.eta_c2, self.eta_c3)


KKT_FIELDS = ("eta_c1", "eta_c2", "eta_c3", "eta_p1", "eta_p2", "eta_p3", "eta_d1", "eta_d2", "eta_gap",
              "obj_primal", "obj_dual")


@dataclass
class SolveResult:
    model: ModelFile
    iterations: int
    psqmr_total: int
    double_count: int
    solve_time: float
    read_time: float
    final_residuals: KKTResiduals
    final_state: SolverState
    train_error_pct: float
    backend_used: SolverKind
    C_used: float
    converged: bool
    # B200 extras (not in the reference record)
    history: Optional[np.ndarray] = None
    setup_ms: float = 0.0
    loop_ms: float = 0.0
    timings: Optional[dict] = None


# ---------------------------------------------------------------------------
# one-time host helpers (solver.py:235-285,343-362)
# ---------------------------------------------------------------------------
def compute_weights(y: np.ndarray, q: float) -> np.ndarray:
    """solver.py:235-250: tau = (n_class / K)^(1/(1+q)), K = n / ln n,
    normalised by the larger; the majority class gets the smaller weight."""
    y = np.asarray(y, dtype=np.float64)
    n = y.size
    if n < 2:
        raise ValueError("need at least two samples")
    n_pos = int(np.sum(y > 0))
    n_neg = int(np.sum(y < 0))
    if n_pos == 0 or n_neg == 0:
        raise SingleClassError("both classes are required to set weights")
    k = n / math.log(n)
    tp = (n_pos / k) ** (1.0 / (1.0 + q))
    tn = (n_neg / k) ** (1.0 / (1.0 + q))
    top = max(tp, tn)
    return np.where(y > 0, tn / top, tp / top)


def scale_problem(x: SparseMatrixCSC, y: np.ndarray, e: Optional[np.ndarray], C: float, q: float,
                  tau: Optional[np.ndarray] = None) -> ProblemData:
    """solver.py:253-285: sign columns by y, divide by sqrt(||X||_F),
    loss weights tau^q."""
    y = np.asarray(y, dtype=np.float64)
    n = x.ncols
    fro = x.frobenius_norm()
    if fro == 0.0:
        raise ValueError("all-zero data matrix")
    z_scale = math.sqrt(fro)
    if x.is_dense:
        vals = (x.dense_samples() * y[:, None]) / z_scale
        z = SparseMatrixCSC.from_dense_samples(vals)
    else:
        col_sign = np.repeat(y, np.diff(x.colptr))
        z = SparseMatrixCSC(x.nrows, x.ncols, x.colptr.copy(), x.rowidx.copy(), x.values * col_sign / z_scale)
    if e is None:
        e = np.ones(n)
    if tau is None:
        tau = np.ones(n)
    weights = np.asarray(tau, dtype=np.float64) ** q
    return ProblemData(z_tilde=z, y=y, e=np.asarray(e, dtype=np.float64), weights=weights, C=float(C),
                       q=float(q), z_scale=z_scale)


def update_sigma(sigma: float, eta_p: float, eta_d: float) -> float:
    """solver.py:343-362 (the device loop applies the same rule)."""
    if eta_p == 0.0 and eta_d == 0.0:
        return sigma
    chi = math.inf if eta_d == 0.0 else eta_p / eta_d
    inv_chi = math.inf if eta_p == 0.0 else eta_d / eta_p
    imbalance = max(chi, inv_chi)
    zeta = 2.2 if imbalance > 500.0 else (1.65 if imbalance > 50.0 else 1.1)
    if chi > 5.0:
        return sigma * zeta
    if inv_chi > 5.0:
        return sigma / zeta
    return sigma


# ---------------------------------------------------------------------------
# device problem handle
# ---------------------------------------------------------------------------
_RAISE = {
    _lib.ERR_VALUE: ValueError,
    _lib.ERR_INDEFINITE: IndefiniteMatrixError,
    _lib.ERR_SCHUR: DegenerateSchurError,
    _lib.ERR_LANCZOS: LanczosConvergenceError,
    _lib.ERR_ASSERT: AssertionError,
    _lib.ERR_UNSUPPORTED: NotImplementedError,
}


def _check(rc: int, ctx=None, what: str = "") -> None:
    if rc == _lib.OK:
        return
    lib = _lib.load()
    msg = lib.gdwd_last_error(ctx).decode() if ctx else ""
    raise _RAISE.get(rc, RuntimeError)(f"{what}: {msg}" if msg else f"{what} failed (code {rc})")


class DeviceProblem:
    """A ProblemData resident in HBM (one gdwd context).

    Z~ is uploaded once; repeated solves on the same ProblemData reuse it and
    the cached factorisation."""

    def __init__(self, data: Optional[ProblemData], device: int = 0, hint: Optional[tuple] = None):
        lib = _lib.load()
        self.lib = lib
        self.device = int(device)
        self.lock = threading.Lock()
        h = C.c_void_p()
        _check(lib.gdwd_ctx_create(self.device, C.byref(h)), None, "gdwd_ctx_create")
        self.ctx = h
        self.n_global = None
        if data is None:  # empty context (device-generated data)
            self.n = self.d = 0
            self.fro = None
            return
        self.n, self.d = data.n, data.d
        z = data.z_tilde
        if z.is_dense:
            vals = z.values
            if hint is not None:  # (backend code, mu) of the coming solve: factor during the upload
                _check(lib.gdwd_upload_hint(self.ctx, int(hint[0]), float(hint[1])), self.ctx, "upload hint")
            _check(lib.gdwd_upload_dense(self.ctx, _lib.ptr(vals), self.d, self.n), self.ctx, "upload")
        else:
            cp = np.ascontiguousarray(z.colptr, dtype=np.int64)
            ri = np.ascontiguousarray(z.rowidx, dtype=np.int64)
            _check(lib.gdwd_upload_csc(self.ctx, cp.ctypes.data_as(C.POINTER(C.c_int64)),
                                       ri.ctypes.data_as(C.POINTER(C.c_int64)), _lib.ptr(_lib.f64(z.values)),
                                       self.d, self.n), self.ctx, "upload")
        _check(lib.gdwd_set_problem(self.ctx, _lib.ptr(_lib.f64(data.y)), _lib.ptr(_lib.f64(data.e)),
                                    _lib.ptr(_lib.f64(data.weights)), float(data.C), float(data.q),
                                    float(data.z_scale)), self.ctx, "set_problem")
        self.fro = None

    def close(self):
        if self.ctx:
            self.lib.gdwd_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def matvec(self, v: np.ndarray) -> np.ndarray:
        v = _lib.f64(v)
        if v.shape != (self.n,):
            raise ValueError(f"dimension mismatch: operand has length {v.shape}, expected ({self.n},)")
        out = np.empty(self.d)
        _check(self.lib.gdwd_matvec(self.ctx, _lib.ptr(v), _lib.ptr(out)), self.ctx, "matvec")
        return out

    def rmatvec(self, v: np.ndarray) -> np.ndarray:
        v = _lib.f64(v)
        if v.shape != (self.d,):
            raise ValueError(f"dimension mismatch: operand has length {v.shape}, expected ({self.d},)")
        out = np.empty(self.n)
        _check(self.lib.gdwd_matvec_t(self.ctx, _lib.ptr(v), _lib.ptr(out)), self.ctx, "matvec_t")
        return out

    def state(self) -> dict:
        n, d = self.n, self.d
        arr = {k: np.empty(n) for k in ("r", "xi", "alpha", "ztw")}
        arr.update({k: np.empty(d) for k in ("w", "u", "rho")})
        b = np.empty(1)
        _check(self.lib.gdwd_get_state(self.ctx, *(_lib.ptr(arr[k]) for k in ("r", "xi", "alpha", "w", "u",
                                                                               "rho", "ztw")), _lib.ptr(b)),
               self.ctx, "get_state")
        arr["beta"] = float(b[0])
        return arr

    def eps_c(self) -> float:
        """1/max(1, ||Z~||_F) from the device-side norm (solver.py:441-445)."""
        fro2 = C.c_double()
        _check(self.lib.gdwd_frobenius_sq(self.ctx, C.byref(fro2)), self.ctx, "frobenius")
        return 1.0 / max(1.0, math.sqrt(fro2.value))

    def history(self, rows: int) -> np.ndarray:
        h = np.zeros((max(rows, 1), 16))
        nr = C.c_int64()
        _check(self.lib.gdwd_get_history(self.ctx, _lib.ptr(h), rows, C.byref(nr)), self.ctx, "get_history")
        return h[: nr.value]


_DEVICE_CACHE: "weakref.WeakValueDictionary[int, DeviceProblem]" = weakref.WeakValueDictionary()


def device_problem(data: ProblemData, device: Optional[int] = None, hint: Optional[tuple] = None) -> DeviceProblem:
    """The (cached) device-resident copy of ``data``.  ``hint`` = (backend
    code, mu) of the solve that follows a first upload."""
    dev = getattr(data, "_gdwd_device", None)
    want = 0 if device is None else int(device)
    if dev is None or dev.ctx is None or dev.device != want:
        dev = DeviceProblem(data, want, hint)
        object.__setattr__(data, "_gdwd_device", dev)
    return dev


def kkt_residuals(state: SolverState, data: ProblemData, mu: float = 1.0) -> KKTResiduals:
    """Normalized optimality residuals of an iterate (solver.py:311-340), on
    the device: one Z~^T w pass with the sample sums, one Z~ alpha pass, one
    d-space map; AssertionError if r left the positive orthant."""
    data = as_problem(data)
    dp = device_problem(data)
    n, d = data.n, data.d
    vec = {k: _lib.f64(getattr(state, k)) for k in ("r", "xi", "alpha", "w", "u")}
    for k, v in vec.items():
        if v.shape != ((n,) if k in ("r", "xi", "alpha") else (d,)):
            raise ValueError(f"dimension mismatch: state.{k} has shape {v.shape}")
    out = np.empty(11)
    _check(dp.lib.gdwd_kkt_residuals(dp.ctx, _lib.ptr(vec["r"]), _lib.ptr(vec["xi"]), _lib.ptr(vec["alpha"]),
                                     _lib.ptr(vec["w"]), _lib.ptr(vec["u"]), float(state.beta), float(mu),
                                     _lib.ptr(out)), dp.ctx, "kkt_residuals")
    return KKTResiduals(*[float(v) for v in out])


def primal_objective(data: ProblemData, r: np.ndarray, xi: np.ndarray) -> float:
    """sum w / r^q + C e.xi (solver.py:306-308), from the device KKT pass."""
    z_n, z_d = np.zeros(data.n), np.zeros(data.d)
    st = SolverState(r, xi, z_n, z_d, z_d, z_d, 0.0, 1.0, 0, 0.0)
    return kkt_residuals(st, data).obj_primal


def dual_objective(data: ProblemData, alpha: np.ndarray) -> float:
    """kappa sum w^(1/(q+1)) max(a,0)^(q/(q+1)) - z_scale ||Z~ a||
    (solver.py:291-303), from the device KKT pass."""
    z_d = np.zeros(data.d)
    st = SolverState(np.ones(data.n), np.zeros(data.n), alpha, z_d, z_d, z_d, 0.0, 1.0, 0, 0.0)
    return kkt_residuals(st, data).obj_dual


def as_problem(data) -> ProblemData:
    """The package's ProblemData for ``data``: itself, a device-generated
    problem (``z_tilde`` is None), or -- drop-in use -- the reference's own
    ``gdwd.ProblemData`` holding a reference ``SparseMatrixCSC`` (solver.py:60-95,
    linalg/sparse.py:20-50), converted once and cached on the object (a fully
    stored CSC becomes the zero-copy dense sample layout)."""
    if isinstance(data, ProblemData) or getattr(data, "z_tilde", 0) is None:
        return data
    cached = getattr(data, "_gdwd_problem", None)
    if cached is not None:
        return cached
    try:
        z = data.z_tilde
        fields = (data.y, data.e, data.weights, data.C, data.q, data.z_scale)
    except AttributeError as exc:
        raise TypeError(f"expected a ProblemData, got {type(data).__name__}") from exc
    out = ProblemData(as_csc(z), *fields)
    try:
        object.__setattr__(data, "_gdwd_problem", out)
    except (AttributeError, TypeError):
        pass
    return out


def _eps_c(data: ProblemData, config: SolverConfig) -> float:
    """solver.py:441-445.  NaN asks the library for the default
    1/max(1, ||Z~||_F), with the norm reduced on the device at upload."""
    if config.epsilon_c is not None:
        return float(config.epsilon_c)
    return float("nan")


# ---------------------------------------------------------------------------
# the solver
# ---------------------------------------------------------------------------
def sgs_admm_solve(data: ProblemData, config: SolverConfig, meta: Optional[FeatureMeta] = None,
                   callback: Optional[Callable[[SolverState, KKTResiduals], None]] = None, *,
                   sigma_schedule: Optional[np.ndarray] = None, device: Optional[int] = None,
                   use_graph: bool = True, poll_every: int = 16, smw_gram_space: bool = True,
                   persistent: bool = True, iter_gram: Optional[bool] = None,
                   devices: Optional[list] = None) -> SolveResult:
    """Run the solver to the KKT stopping rule or the iteration cap
    (solver.py:392-602).  ``callback(state, residuals)`` runs after every
    iteration (it forces a device sync and a copy of the iterates).

    Keyword-only B200 extras: ``sigma_schedule`` (test hook: sigma of
    iteration k replaces update_sigma for 1 <= k < len), ``device``,
    ``use_graph``, ``poll_every``, ``smw_gram_space`` (SMW2 regime: iterate
    in sample-coefficient space with the n x n Gram instead of passes over X),
    ``persistent`` (Gram-space SMW2: all iterations in one cooperative kernel),
    ``iter_gram`` (ITERATIVE on dense data: PSQMR's operator from the d x d
    Gram formed once on the FP64 tensor cores; None = automatic for d <= n/4),
    ``devices`` (a list of GPUs: the samples are sharded over them from this
    one process, parallel.solve_on_devices)."""
    if devices is not None and len(devices) > 1:
        from .parallel import solve_on_devices

        return solve_on_devices(data, config, devices, meta=meta, callback=callback, sigma_schedule=sigma_schedule,
                                use_graph=use_graph, poll_every=poll_every, smw_gram_space=smw_gram_space,
                                persistent=persistent, iter_gram=iter_gram)
    if devices is not None and len(devices) == 1:
        device = int(devices[0])
    t_start = time.perf_counter()
    data = as_problem(data)
    hint = None
    if getattr(data, "_gdwd_device", None) is None and data.z_tilde is not None:
        hint = (_lib.BACKEND_CODE[config.backend.resolve(data.n, data.d).value], config.mu)
    dp = device_problem(data, device, hint)
    t_up = time.perf_counter()
    lib = dp.lib
    kind = config.backend.resolve(dp.n_global or data.n, data.d)  # sharded: the global sample count
    eps_c = _eps_c(data, config)
    cfg = _lib.GdwdConfig(
        max_iter=int(config.max_iter), backend=_lib.BACKEND_CODE[kind.value], use_sgs=int(bool(config.use_sgs)),
        psqmr_switch_steps=int(config.psqmr_switch_steps), ell=int(config.ell), seed=int(config.seed),
        use_graph=int(bool(use_graph)), poll_every=int(poll_every), smw_gram_space=int(bool(smw_gram_space)),
        persistent=int(bool(persistent)), iter_gram=0 if iter_gram is None else (1 if iter_gram else -1),
        steplength=float(config.steplength),
        tol_feas=float(config.tol_feas), tol_cgap=float(config.tol_cgap), tol_cap=float(config.tol_cap),
        sigma0=float("nan") if config.sigma0 is None else float(config.sigma0), epsilon_c=eps_c,
        mu=float(config.mu))
    sched = None if sigma_schedule is None else _lib.f64(sigma_schedule)
    if kind is SolverKind.ITERATIVE:
        # start vector of the proximal fallback's Lanczos run (lanczos.py:85)
        v0 = np.random.default_rng(config.seed).standard_normal(data.d)
        _check(lib.gdwd_set_lanczos_start(dp.ctx, _lib.ptr(v0), data.d), dp.ctx, "lanczos start")
    err: list = []

    def _cb(user, it, resid_p, sigma, beta):
        try:
            st = dp.state()
            res = KKTResiduals(*[float(resid_p[i]) for i in range(11)])
            state = SolverState(st["r"], st["xi"], st["alpha"], st["w"], st["u"], st["rho"], float(beta),
                                float(sigma), int(it), eps_c if eps_c == eps_c else dp.eps_c())
            callback(state, res)
            return 0
        except BaseException as exc:  # propagate after the C call returns
            err.append(exc)
            return 1

    cfun = _lib.ITER_CB(_cb) if callback is not None else _lib.ITER_CB()
    out = _lib.GdwdResult()
    with dp.lock:
        rc = lib.gdwd_solve(dp.ctx, C.byref(cfg), _lib.ptr(sched), 0 if sched is None else sched.size, cfun, None,
                            C.byref(out))
        if rc == _lib.ERR_ABORTED and err:
            raise err[0]
        _check(rc, dp.ctx, "gdwd_solve")
        t_solved = time.perf_counter()
        st = dp.state()
        hist = dp.history(out.iterations)
    solve_time = time.perf_counter() - t_start
    resid = KKTResiduals(*[float(out.resid[i]) for i in range(11)])
    sigma_last = float(hist[-1, 11]) if len(hist) else float(out.sigma)
    state = SolverState(st["r"], st["xi"], st["alpha"], st["w"], st["u"], st["rho"], st["beta"], sigma_last,
                        int(out.iterations), float(out.eps_c))
    # train error over ALL samples (solver.py:557-559): a sharded rank counts
    # its own misclassified samples and the counts are summed over the shards
    scores = st["beta"] + data.y * st["ztw"]
    bad = np.array([float(np.sum(data.y * np.sign(scores) <= 0.0))])
    if dp.n_global:
        _check(lib.gdwd_allreduce_host(dp.ctx, _lib.ptr(bad), 1), dp.ctx, "train error all-reduce")
    train_err = 100.0 * (float(bad[0]) / float(dp.n_global or data.n))
    if meta is None:
        meta = identity_meta(data.d)
    converged = bool(out.converged)
    model = ModelFile(
        q=data.q, C=data.C, z_scale=data.z_scale, mu=config.mu, feature_meta=meta, w=st["w"] / data.z_scale,
        beta=st["beta"],
        solver_info={
            "iterations": int(out.iterations), "converged": converged, "backend": kind.value,
            "psqmr_total": int(out.psqmr_total), "double_count": int(out.double_count),
            "solve_time": solve_time, "train_error_pct": train_err,
            "residuals": {"eta_p": resid.eta_p, "eta_d": resid.eta_d, "eta_c": resid.eta_c,
                          "eta_gap": resid.eta_gap, "obj_primal": resid.obj_primal, "obj_dual": resid.obj_dual},
        })
    return SolveResult(model=model, iterations=int(out.iterations), psqmr_total=int(out.psqmr_total),
                       double_count=int(out.double_count), solve_time=solve_time, read_time=0.0,
                       final_residuals=resid, final_state=state, train_error_pct=train_err, backend_used=kind,
                       C_used=data.C, converged=converged, history=hist, setup_ms=float(out.setup_ms),
                       loop_ms=float(out.loop_ms),
                       timings={"upload_s": t_up - t_start, "solve_call_s": t_solved - t_up,
                                "download_s": solve_time - (t_solved - t_start), "setup_ms": float(out.setup_ms),
                                "loop_ms": float(out.loop_ms)})


# ---------------------------------------------------------------------------
# subsolver seams on the device
# ---------------------------------------------------------------------------
def newton_r_sweep(a, sigma: float, q: float, weights, r_init, tol: float, max_newton: int = 50,
                   device: int = 0) -> np.ndarray:
    """subsolvers.py:321-364 on the device."""
    a = _lib.f64(a)
    w = _lib.f64(weights)
    r0 = _lib.f64(r_init)
    out = np.empty_like(a)
    lib = _lib.load()
    _check(lib.gdwd_newton_sweep(device, a.size, _lib.ptr(a), float(sigma), float(q), _lib.ptr(w), _lib.ptr(r0),
                                 float(tol), int(max_newton), 0, _lib.ptr(out), None), None, "newton_r_sweep")
    return out


def newton_r(a: float, sigma: float, q: float, weight: float, r_init: float, tol: float = 1e-12,
             max_newton: int = 50, device: int = 0) -> tuple[float, int]:
    """subsolvers.py:283-318 (scalar; returns (root, newton iterations))."""
    if sigma <= 0 or q <= 0 or weight <= 0 or r_init <= 0:
        raise ValueError("sigma, q, weight and r_init must be positive")
    lib = _lib.load()
    out = np.empty(1)
    it = (C.c_int32 * 1)()
    _check(lib.gdwd_newton_sweep(device, 1, _lib.ptr(np.array([a], float)), float(sigma), float(q),
                                 _lib.ptr(np.array([weight], float)), _lib.ptr(np.array([r_init], float)),
                                 float(tol), int(max_newton), 1, _lib.ptr(out), it), None, "newton_r")
    return float(out[0]), int(it[0])


def matvec(m: SparseMatrixCSC, x: np.ndarray, transpose: bool = False, device: int = 0) -> np.ndarray:
    """linalg/sparse.py:129-142 on the device (dense or sparse CSC storage)."""
    x = _lib.f64(x)
    expected = m.nrows if transpose else m.ncols
    if x.shape != (expected,):
        raise ValueError(f"dimension mismatch: operand has length {x.shape}, expected ({expected},)")
    ones = np.ones(m.ncols)
    pd = ProblemData(m, ones, ones, ones, 1.0, 1.0, 1.0)
    dp = DeviceProblem(pd, device)
    try:
        return dp.rmatvec(x) if transpose else dp.matvec(x)
    finally:
        dp.close()


__all__ = ["Backend", "DegenerateSchurError", "DeviceProblem", "IndefiniteMatrixError", "KKTResiduals",
           "KKT_FIELDS", "LanczosConvergenceError", "ProblemData", "SingleClassError", "SolveResult",
           "SolverConfig", "SolverKind", "SolverState", "as_problem", "compute_weights", "device_problem", "matvec",
           "newton_r", "newton_r_sweep", "scale_problem", "select_solver", "sgs_admm_solve", "update_sigma"]
