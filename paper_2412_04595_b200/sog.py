"""ctypes binding of libsog.so (include/sog.h).  Argument marshalling only."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

SOG_NO_VALIDATE = 1
SOG_TIMING = 2
SOG_GRAPH = 4
STATUS = {0: "SOG_OK", -1: "SOG_EINVAL", -2: "SOG_ENONNEUTRAL", -3: "SOG_EZRANGE",
          -4: "SOG_ENONFINITE", -5: "SOG_EINFEASIBLE", -6: "SOG_ECUDA", -7: "SOG_ENCCL", -8: "SOG_ENOMEM"}
TIMING_NAMES = ["sort", "near", "mid_spread", "mid_fft_fwd", "mid_scale", "mid_fft_inv", "mid_gather",
                "long_spread", "long_fft_scale_ifft", "long_gather", "combine"]
EXPORTS = ["sog_plan_create", "sog_plan_choose", "sog_plan_create_ex", "sog_eval", "sog_eval_host", "sog_eval_host_async",
           "sog_host_wait", "sog_eval_components",
           "sog_debug_stage", "sog_last_energy", "sog_plan_destroy", "sog_last_error", "sog_plan_describe",
           "sog_get_timings", "sog_set_flags", "sog_set_stream", "sog_launches_per_eval",
           "sog_nccl_selftest", "sog_nccl_unique_id", "sog_dist_create", "sog_dist_create_loopback", "sog_dist_eval",
           "sog_dist_local_ranks", "sog_dist_describe", "sog_dist_destroy", "sog_dist_set_flags",
           "sog_dist_get_timings"]


class SogError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class Opts(ctypes.Structure):
    _fields_ = [("rc_factor", ctypes.c_double), ("eta", ctypes.c_double),
                ("explicit_params", ctypes.c_int), ("row", ctypes.c_int), ("rc", ctypes.c_double),
                ("M", ctypes.c_int), ("m", ctypes.c_int),
                ("Ix", ctypes.c_int), ("Iy", ctypes.c_int), ("Iz", ctypes.c_int), ("Izs", ctypes.c_int),
                ("P", ctypes.c_int), ("S", ctypes.c_double),
                ("Ilx", ctypes.c_int), ("Ily", ctypes.c_int), ("Pl", ctypes.c_int), ("Sl", ctypes.c_double),
                ("Pc", ctypes.c_int), ("cuda_stream", ctypes.c_void_p), ("flags", ctypes.c_uint),
                ("precision", ctypes.c_int), ("window", ctypes.c_int), ("nu", ctypes.c_int),
                ("nul", ctypes.c_int), ("long_method", ctypes.c_int), ("Kx", ctypes.c_int), ("Ky", ctypes.c_int),
                ("optimize", ctypes.c_int), ("b", ctypes.c_double), ("r0", ctypes.c_double),
                ("omega", ctypes.c_double)]

WINDOWS = {"gs": 0, "kb": 1, "es": 2}
LONG_METHODS = {"fft": 0, "direct": 1}


def _set_window(o, window, params, long_method="fft"):
    """Window / long-range method: explicit params carry their own (oracle Plan: "gs"/"kb",
    "fft"/"direct"), else the keyword arguments."""
    w = params.get("window", window) if params is not None else window
    o.window = WINDOWS[w] if isinstance(w, str) else int(w)
    lm = params.get("long_method", long_method) if params is not None else long_method
    o.long_method = LONG_METHODS[lm] if isinstance(lm, str) else int(lm)
    if params is not None:
        o.nu = int(params.get("nu", 0))
        o.nul = int(params.get("nul", 0))
        o.Kx = int(params.get("Kx", 0))
        o.Ky = int(params.get("Ky", 0))


def lib_path() -> str:
    # SOG_LIB: another in-tree build of the same library under lib/ (A/B measurements of kernel
    # variants, scripts/gpu_ab_libs.sh); nothing outside the package's lib/ directory is loaded
    lib_dir = os.path.join(HERE, "lib")
    alt = os.environ.get("SOG_LIB")
    if alt:
        alt = os.path.realpath(alt if os.path.isabs(alt) else os.path.join(lib_dir, alt))
        if os.path.dirname(alt) != os.path.realpath(lib_dir):
            raise ImportError(f"SOG_LIB={alt}: only builds in {lib_dir} can be loaded")
        return alt
    return os.path.join(lib_dir, "libsog.so")


def load_library():
    """Load the in-tree libsog.so (raises if it has not been built: no fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = lib_path()
    if not os.path.exists(path):
        raise ImportError(f"{path} missing: run `python -m paper_2412_04595_b200.build` (no CPU fallback)")
    lib = ctypes.CDLL(path)
    P, D, I, U, S = ctypes.c_void_p, ctypes.c_double, ctypes.c_int, ctypes.c_uint, ctypes.c_size_t
    lib.sog_plan_create.restype = P
    lib.sog_plan_create.argtypes = [ctypes.c_int64, D, D, D, D]
    lib.sog_plan_choose.restype = I
    lib.sog_plan_choose.argtypes = [ctypes.c_int64, D, D, D, D, ctypes.POINTER(Opts), ctypes.c_char_p, S]
    lib.sog_plan_create_ex.restype = P
    lib.sog_plan_create_ex.argtypes = [ctypes.c_int64, D, D, D, D, ctypes.POINTER(Opts)]
    for name in ("sog_eval", "sog_eval_host", "sog_eval_host_async"):
        getattr(lib, name).restype = I
        getattr(lib, name).argtypes = [P, P, P, P, P]
    lib.sog_host_wait.restype = I
    lib.sog_host_wait.argtypes = [P]
    lib.sog_eval_components.restype = I
    lib.sog_eval_components.argtypes = [P, P, P, P]
    lib.sog_debug_stage.restype = I
    lib.sog_debug_stage.argtypes = [P, I, P, P, P, S]
    lib.sog_last_energy.restype = I
    lib.sog_last_energy.argtypes = [P, ctypes.POINTER(D)]
    lib.sog_plan_destroy.restype = None
    lib.sog_plan_destroy.argtypes = [P]
    lib.sog_last_error.restype = ctypes.c_char_p
    lib.sog_last_error.argtypes = []
    lib.sog_plan_describe.restype = I
    lib.sog_plan_describe.argtypes = [P, ctypes.c_char_p, S]
    lib.sog_get_timings.restype = I
    lib.sog_get_timings.argtypes = [P, ctypes.POINTER(D), I]
    lib.sog_set_flags.restype = I
    lib.sog_set_flags.argtypes = [P, U]
    lib.sog_set_stream.restype = I
    lib.sog_set_stream.argtypes = [P, P]
    lib.sog_launches_per_eval.restype = I
    lib.sog_launches_per_eval.argtypes = [P]
    I64 = ctypes.c_int64
    lib.sog_nccl_unique_id.restype = I
    lib.sog_nccl_unique_id.argtypes = [P]
    lib.sog_dist_create.restype = P
    lib.sog_dist_create.argtypes = [I64, I64, D, D, D, D, ctypes.POINTER(Opts), I, I, P]
    lib.sog_dist_create_loopback.restype = P
    lib.sog_dist_create_loopback.argtypes = [I64, I64, D, D, D, D, ctypes.POINTER(Opts), I]
    lib.sog_dist_eval.restype = I
    lib.sog_dist_eval.argtypes = [P, P, P, P, P, P]
    lib.sog_dist_local_ranks.restype = I
    lib.sog_dist_local_ranks.argtypes = [P]
    lib.sog_dist_describe.restype = I
    lib.sog_dist_describe.argtypes = [P, ctypes.c_char_p, S]
    lib.sog_dist_destroy.restype = None
    lib.sog_dist_destroy.argtypes = [P]
    lib.sog_dist_set_flags.restype = I
    lib.sog_dist_set_flags.argtypes = [P, U]
    lib.sog_dist_get_timings.restype = I
    lib.sog_dist_get_timings.argtypes = [P, ctypes.POINTER(D), I]
    _LIB = lib
    return lib


def _err(lib, code):
    return SogError(code, lib.sog_last_error().decode())


PLAN_FIELDS = ("row", "rc", "M", "m", "Ix", "Iy", "Iz", "Izs", "P", "S", "Ilx", "Ily", "Pl", "Sl", "Pc")


class Plan:
    """A solver plan for N charges in the box L = (Lx, Ly, Lz) at tolerance tol.

    params: optional dict with every PLAN_FIELDS entry -> used verbatim (explicit plan);
    rc_factor / eta: overrides of rules R2 / R4;  stream: torch.cuda.Stream or raw handle.
    """

    def __init__(self, N, L, tol, params=None, rc_factor=None, eta=None, stream=None,
                 validate=True, timing=False, precision="fp64", window="gs", long_method="fft", optimize=False,
                 b=None):
        """b: a general SOG base in (1, 2] (NEXT #4: (r0, omega) by the C^1 solve) instead of R1's row."""
        self.lib = load_library()
        self.N = int(N)
        self.L = tuple(float(v) for v in L)
        self.tol = float(tol)
        o = Opts()
        o.rc_factor = float(rc_factor or 0.0)
        o.eta = float(eta or 0.0)
        if params is not None:
            o.explicit_params = 1
            for k in PLAN_FIELDS:
                setattr(o, k, type(getattr(o, k))(params[k]))
            if params.get("row", 0) is None or int(params.get("row", 0)) < 0:   # general b (NEXT #4)
                o.b, o.r0, o.omega = float(params["b"]), float(params["r0"]), float(params["omega"])
                o.row = -1
        elif b is not None:
            o.b = float(b)
        o.flags = (0 if validate else SOG_NO_VALIDATE) | (SOG_TIMING if timing else 0)
        o.cuda_stream = _stream_handle(stream)
        o.precision = {"fp64": 0, "fp32": 1}[precision]
        _set_window(o, window, params, long_method)
        o.optimize = int(bool(optimize))
        h = self.lib.sog_plan_create_ex(self.N, *self.L, self.tol, ctypes.byref(o))
        if not h:
            raise SogError(-1, self.lib.sog_last_error().decode())
        self.h = h
        self._flags = o.flags

    # -- lifecycle
    def close(self):
        if getattr(self, "h", None):
            self.lib.sog_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- configuration
    def describe(self) -> dict:
        n = self.lib.sog_plan_describe(self.h, None, 0)
        buf = ctypes.create_string_buffer(n + 1)
        self.lib.sog_plan_describe(self.h, buf, n + 1)
        return _parse(buf.value.decode())

    def set_flags(self, validate=True, timing=False, graph=False):
        """graph=True: replay the evaluation as one CUDA graph (SOG_GRAPH; no stage timings)."""
        self._flags = (0 if validate else SOG_NO_VALIDATE) | (SOG_TIMING if timing else 0) | (SOG_GRAPH if graph else 0)
        self._check(self.lib.sog_set_flags(self.h, self._flags))

    def set_stream(self, stream):
        self._check(self.lib.sog_set_stream(self.h, _stream_handle(stream)))

    def launches_per_eval(self) -> int:
        return self.lib.sog_launches_per_eval(self.h)

    def timings(self) -> dict:
        arr = (ctypes.c_double * 11)()
        n = self.lib.sog_get_timings(self.h, arr, 11)
        return {TIMING_NAMES[i]: arr[i] for i in range(n)}

    def energy(self) -> float:
        u = ctypes.c_double()
        self._check(self.lib.sog_last_energy(self.h, ctypes.byref(u)))
        return u.value

    def _check(self, rc):
        if rc != 0:
            raise _err(self.lib, rc)

    # -- evaluation (device tensors)
    def _inputs(self, xyz, q):
        import torch
        if not (xyz.is_cuda and q.is_cuda):
            raise ValueError("xyz and q must be CUDA tensors (use eval_host for host arrays)")
        if xyz.dtype != torch.float64 or q.dtype != torch.float64:
            raise ValueError("xyz and q must be float64")
        if tuple(xyz.shape) != (self.N, 3) or tuple(q.shape) != (self.N,):
            raise ValueError(f"expected xyz [{self.N},3] and q [{self.N}]")
        return xyz.contiguous(), q.contiguous()

    def eval(self, xyz, q, phi=None, force=None, want_force=True):
        """phi [N], force [N,3] (float64 CUDA tensors) for device inputs."""
        import torch
        xyz, q = self._inputs(xyz, q)
        if phi is None:
            phi = torch.empty(self.N, dtype=torch.float64, device=xyz.device)
        if force is None and want_force:
            force = torch.empty(self.N, 3, dtype=torch.float64, device=xyz.device)
        _check_out(phi, (self.N,), xyz.device, "phi")
        if force is not None:
            _check_out(force, (self.N, 3), xyz.device, "force")
        self._check(self.lib.sog_eval(self.h, xyz.data_ptr(), q.data_ptr(), phi.data_ptr(),
                                      force.data_ptr() if force is not None else None))
        return phi, force

    def eval_host(self, xyz, q, phi=None, force=None):
        """Host-buffer path (sog_eval_host): numpy or (pinned) CPU torch arrays in, host arrays out."""
        import numpy as np
        for a, shape, name in ((xyz, (self.N, 3), "xyz"), (q, (self.N,), "q")):
            if tuple(a.shape) != shape:
                raise ValueError(f"{name} must have shape {shape}")
        xyz_p, q_p = _host_ptr(xyz), _host_ptr(q)
        if phi is None:
            phi = np.empty(self.N, dtype=np.float64)
        if force is None:
            force = np.empty((self.N, 3), dtype=np.float64)
        for a, shape, name in ((phi, (self.N,), "phi"), (force, (self.N, 3), "force")):
            if tuple(a.shape) != shape:
                raise ValueError(f"{name} must have shape {shape}")
        self._check(self.lib.sog_eval_host(self.h, xyz_p, q_p, _host_ptr(phi), _host_ptr(force)))
        return phi, force

    def eval_host_async(self, xyz, q, phi, force):
        """Pipelined host-buffer path (sog_eval_host_async): enqueue and return; results are in phi /
        force (host arrays, pinned CPU tensors for asynchronous copies) after host_wait().  The
        arrays must stay alive and the inputs unmodified until then."""
        for a, shape, name in ((xyz, (self.N, 3), "xyz"), (q, (self.N,), "q"), (phi, (self.N,), "phi"),
                               (force, (self.N, 3), "force")):
            if tuple(a.shape) != shape:
                raise ValueError(f"{name} must have shape {shape}")
        self._pending = getattr(self, "_pending", []) + [(xyz, q, phi, force)]
        self._check(self.lib.sog_eval_host_async(self.h, _host_ptr(xyz), _host_ptr(q), _host_ptr(phi),
                                                 _host_ptr(force)))

    def host_wait(self):
        """Wait for every pending eval_host_async call."""
        try:
            self._check(self.lib.sog_host_wait(self.h))
        finally:
            self._pending = []

    def components(self, xyz, q):
        """[3, N, 4] tensor: near / mid / long (phi, dphi/dx, dphi/dy, dphi/dz), self term not removed."""
        import torch
        xyz, q = self._inputs(xyz, q)
        out = torch.empty(3, self.N, 4, dtype=torch.float64, device=xyz.device)
        self._check(self.lib.sog_eval_components(self.h, xyz.data_ptr(), q.data_ptr(), out.data_ptr()))
        return out

    def debug_stage(self, stage, xyz, q):
        """Intermediate grid (1: mid spread, 2: mid Psi, both [Izs][Ix][Iy]; 3: long proxies,
        4: long Psi, both [Pc][Ilx][Ily]) -- the library's device layouts, unchanged."""
        import torch
        d = self.describe()
        if stage in (1, 2):
            shape = (d["Izs"], d["Ix"], d["Iy"])
        else:
            shape = (d["Pc"], d["Ilx"], d["Ily"])
        xyz, q = self._inputs(xyz, q)
        out = torch.empty(shape, dtype=torch.float64, device=xyz.device)
        self._check(self.lib.sog_debug_stage(self.h, stage, xyz.data_ptr(), q.data_ptr(), out.data_ptr(),
                                             out.numel()))
        return out


def _parse(text):
    out = {}
    for line in text.splitlines():
        k, v = line.split("=", 1)
        try:
            out[k] = int(v)
        except ValueError:
            out[k] = float(v)
    return out


def choose_params(N, L, tol, rc_factor=None, eta=None, window="gs", long_method="fft", optimize=False,
                  b=None) -> dict:
    """Plan parameters chosen by the library's rules R1-R9 (host only, no GPU); b: a general SOG
    base (NEXT #4, C^1 solve) instead of R1's Table-1 row."""
    lib = load_library()
    o = Opts()
    if b is not None:
        o.b = float(b)
    o.rc_factor = float(rc_factor or 0.0)
    o.eta = float(eta or 0.0)
    _set_window(o, window, None, long_method)
    o.optimize = int(bool(optimize))
    n = lib.sog_plan_choose(int(N), *[float(v) for v in L], float(tol), ctypes.byref(o), None, 0)
    if n < 0:
        raise _err(lib, n)
    buf = ctypes.create_string_buffer(n + 1)
    lib.sog_plan_choose(int(N), *[float(v) for v in L], float(tol), ctypes.byref(o), buf, n + 1)
    return _parse(buf.value.decode())


def _check_out(t, shape, device, name):
    """Caller-supplied output tensors: the library writes 8 bytes x prod(shape) through the pointer."""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.device != device:
        raise ValueError(f"{name} must be a CUDA tensor on {device}")
    if t.dtype != torch.float64 or tuple(t.shape) != tuple(shape) or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous float64 tensor of shape {tuple(shape)}")


def _check_in(x, shape, name):
    import torch
    if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dtype != torch.float64 or tuple(x.shape) != tuple(shape):
        raise ValueError(f"{name} must be a float64 CUDA tensor of shape {tuple(shape)}")


def _stream_handle(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return getattr(stream, "cuda_stream", None)


def _host_ptr(a):
    import numpy as np
    if isinstance(a, np.ndarray):
        if a.dtype != np.float64 or not a.flags.c_contiguous:
            raise ValueError("host arrays must be C-contiguous float64")
        return a.ctypes.data
    # torch CPU tensor
    import torch
    if a.is_cuda or not a.is_contiguous() or a.dtype != torch.float64:
        raise ValueError("host tensors must be contiguous float64 CPU tensors")
    return a.data_ptr()


def slab_owner(x, Lx, R):
    """Rank owning canonical x under the x-slab rule of include/sog.h (host-side helper, numpy)."""
    import numpy as np
    x = np.asarray(x, dtype=np.float64)
    xc = x - Lx * np.floor((x + 0.5 * Lx) / Lx)
    xc = np.where(xc >= 0.5 * Lx, xc - Lx, xc)
    r = np.floor((xc + 0.5 * Lx) * R / Lx).astype(np.int64)
    # the library's slab edges are -Lx/2 + r Lx / R evaluated in fp64: settle ties exactly
    lo = -0.5 * Lx + Lx * r / R
    r = np.where(xc < lo, r - 1, r)
    hi = np.where(r + 1 == R, 0.5 * Lx, -0.5 * Lx + Lx * (r + 1) / R)
    r = np.where(xc >= hi, r + 1, r)
    return np.clip(r, 0, R - 1)


class DistPlan:
    """x-slab decomposition over R ranks (include/sog.h).

    loopback=True: all R ranks as virtual ranks of this process on the current GPU;
    eval() then takes lists of per-rank tensors.  loopback=False: one rank per process over
    NCCL; pass rank, nranks and the 128-byte NCCL id (see nccl_unique_id / from_process_group).
    """

    def __init__(self, N_total, n_own_max, L, tol, R, rank=0, nccl_id=None, loopback=False, params=None,
                 stream=None, window="gs", validate=True):
        """validate=False skips the invalid-input checks (non-finite, z range, neutrality); slab
        membership and capacities are always checked, identically on every rank."""
        self.lib = load_library()
        self.L = tuple(float(v) for v in L)
        self.R = int(R)
        o = Opts()
        if params is not None:
            o.explicit_params = 1
            for k in PLAN_FIELDS:
                setattr(o, k, type(getattr(o, k))(params[k]))
        o.flags = 0 if validate else SOG_NO_VALIDATE
        o.cuda_stream = _stream_handle(stream)
        _set_window(o, window, params)
        if loopback:
            h = self.lib.sog_dist_create_loopback(int(N_total), int(n_own_max), *self.L, float(tol), ctypes.byref(o),
                                                  self.R)
        else:
            buf = ctypes.create_string_buffer(bytes(nccl_id), 128)
            h = self.lib.sog_dist_create(int(N_total), int(n_own_max), *self.L, float(tol), ctypes.byref(o),
                                         int(rank), self.R, buf)
        if not h:
            raise SogError(-1, self.lib.sog_last_error().decode())
        self.h = h
        self.nlocal = self.lib.sog_dist_local_ranks(h)

    @staticmethod
    def nccl_unique_id() -> bytes:
        lib = load_library()
        buf = ctypes.create_string_buffer(128)
        rc = lib.sog_nccl_unique_id(buf)
        if rc:
            raise _err(lib, rc)
        return buf.raw

    @classmethod
    def from_process_group(cls, N_total, n_own_max, L, tol, **kw):
        """One rank per process: the NCCL id is created on rank 0 and broadcast with torch.distributed."""
        import torch.distributed as dist
        rank, R = dist.get_rank(), dist.get_world_size()
        obj = [cls.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return cls(N_total, n_own_max, L, tol, R, rank=rank, nccl_id=obj[0], **kw)

    DIST_TIMING_NAMES = ("halo", "sort", "mid_spread_fft2d", "a2a_fwd", "xfft_scale", "a2a_bwd", "fft2d_inv",
                         "psi_halo", "gather_long_spread", "long_allreduce", "long_rest", "near")

    def set_flags(self, validate=True, timing=False):
        rc = self.lib.sog_dist_set_flags(self.h, (0 if validate else SOG_NO_VALIDATE) | (SOG_TIMING if timing else 0))
        if rc:
            raise _err(self.lib, rc)

    def timings(self) -> dict:
        arr = (ctypes.c_double * 12)()
        n = self.lib.sog_dist_get_timings(self.h, arr, 12)
        return {self.DIST_TIMING_NAMES[i]: arr[i] for i in range(n)}

    def describe(self) -> dict:
        n = self.lib.sog_dist_describe(self.h, None, 0)
        buf = ctypes.create_string_buffer(n + 1)
        self.lib.sog_dist_describe(self.h, buf, n + 1)
        return _parse(buf.value.decode())

    def eval(self, xyz, q, phi=None, force=None):
        """xyz, q: (lists of, for loopback) CUDA float64 tensors of this rank's own particles."""
        import torch
        single = not isinstance(xyz, (list, tuple))
        xs, qs = ([xyz], [q]) if single else (list(xyz), list(q))
        if len(xs) != self.nlocal:
            raise ValueError(f"expected {self.nlocal} per-rank inputs")
        xs = [x.contiguous() for x in xs]
        qs = [v.contiguous() for v in qs]
        for x, v in zip(xs, qs):
            if v.dim() != 1:
                raise ValueError("q must be one-dimensional")
            _check_in(v, (len(v),), "q")
            _check_in(x, (len(v), 3), "xyz")
            if x.device != v.device:
                raise ValueError("xyz and q of a rank must be on the same device")
        phis = [torch.empty(len(v), dtype=torch.float64, device=v.device) for v in qs] if phi is None else (
            [phi] if single else list(phi))
        fs = [torch.empty(len(v), 3, dtype=torch.float64, device=v.device) for v in qs] if force is None else (
            [force] if single else list(force))
        if len(phis) != self.nlocal or len(fs) != self.nlocal:
            raise ValueError(f"expected {self.nlocal} per-rank outputs")
        for v, ph, f in zip(qs, phis, fs):
            _check_out(ph, (len(v),), v.device, "phi")
            _check_out(f, (len(v), 3), v.device, "force")
        n = (ctypes.c_int64 * self.nlocal)(*[len(v) for v in qs])
        P = ctypes.c_void_p * self.nlocal
        rc = self.lib.sog_dist_eval(self.h, n, P(*[x.data_ptr() for x in xs]), P(*[v.data_ptr() for v in qs]),
                                    P(*[v.data_ptr() for v in phis]), P(*[v.data_ptr() for v in fs]))
        if rc:
            raise _err(self.lib, rc)
        return (phis[0], fs[0]) if single else (phis, fs)

    def close(self):
        if getattr(self, "h", None):
            self.lib.sog_dist_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def redistribute(xyz, q, L, group=None):
    """Move every particle to the rank owning its x slab (torch.distributed, any backend):
    returns this rank's (xyz, q, origin) where origin = (source rank, source index) per
    particle, so results can be sent back.  Host-side marshalling for sog_dist_eval."""
    import torch
    import torch.distributed as dist
    R, me = dist.get_world_size(group), dist.get_rank(group)
    dev = xyz.device
    owner = torch.from_numpy(slab_owner(xyz[:, 0].detach().cpu().numpy(), float(L[0]), R)).to(dev)
    order = torch.argsort(owner, stable=True)
    counts = torch.bincount(owner, minlength=R)
    rcounts = torch.empty_like(counts)
    dist.all_to_all_single(rcounts, counts, group=group)
    sc, rc = counts.tolist(), rcounts.tolist()
    idx = torch.arange(len(q), device=dev, dtype=torch.float64)
    rank_col = torch.full((len(q),), float(me), device=dev, dtype=torch.float64)
    send = torch.cat([xyz, q[:, None], rank_col[:, None], idx[:, None]], dim=1)[order].contiguous()
    recv = torch.empty(sum(rc), 6, dtype=torch.float64, device=dev)
    dist.all_to_all_single(recv, send, output_split_sizes=rc, input_split_sizes=sc, group=group)
    return recv[:, :3].contiguous(), recv[:, 3].contiguous(), recv[:, 4:].to(torch.int64)
