"""ctypes binding of libtm.so (names follow include/tm.h; marshalling only)."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libtm.so")

TM_I8, TM_F32 = 0, 1
TM_BINARY = 1
TM_CORR_NTT, TM_CORR_TC = 2, 4
TM_ALIAS_REPAIR = 8
TM_BLOCK = 16
TM_INPUTS_STABLE = 32
TM_KEEP_Y = 64
_ENGINES = {None: 0, "auto": 0, "ntt": TM_CORR_NTT, "tc": TM_CORR_TC}
TM_OK, TM_EINVAL, TM_EUNSUPPORTED, TM_ECUDA = 0, 1, 2, 3

EXPORTED_SYMBOLS = (
    "tm_plan_create", "tm_plan_query", "tm_workspace_bytes", "tm_plan_destroy", "tm_generate",
    "tm_fold", "tm_fold_template", "tm_correlate", "tm_match", "tm_run", "tm_run_host", "tm_correlate_match", "tm_correlate_many",
    "tm_status_string", "tm_last_error", "tm_launch_count", "tm_profile_events", "tm_run_path",
    "tm_correlate_match_part", "tm_match_keys",
    "tm_mplan_create", "tm_mplan_workspace_bytes", "tm_mplan_run", "tm_crt_multi", "tm_mplan_destroy",
    "tm_run_fold_rows", "tm_probe_read_bw", "tm_probe_read_pattern", "tm_fold_reduce",
)
RUN_PATHS = {0: "staged (fold -> NTT/fp32 correlation -> CRT)", 1: "staged (fold -> tensor-core correlation)",
             2: "fused (fold + tensor-core correlation in one kernel)", 3: "small pair (whole path, one CTA per pair)"}

_i64, _u64, _i32, _u32, _p, _d = (ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, ctypes.c_uint32,
                                  ctypes.c_void_p, ctypes.c_double)


class PlanInfo(ctypes.Structure):
    _fields_ = [("N", _i64), ("K", _i64), ("M1", _i64), ("M2", _i64), ("q1", _i64), ("q2", _i64),
                ("s1", _i64), ("s2", _i64), ("len_y1", _i64), ("len_y2", _i64), ("L1", _i64),
                ("L2", _i64), ("n_primes", _i32), ("dtype", _i32), ("flags", _u32),
                ("fast_fold", _i32), ("tf_bytes", _i64), ("seed", _u64),
                ("corr_engine", _i32)]


class TMError(RuntimeError):
    def __init__(self, status: int, where: str):
        L = lib()
        msg = L.tm_last_error().decode(errors="replace")
        name = L.tm_status_string(status).decode()
        super().__init__(f"{where}: {name}: {msg}")
        self.status = status


_lib = None


def lib_path() -> str:
    # TM_LIB_VARIANT=<name> loads paper_1509_04863_b200/libtm_<name>.so instead
    # (same-box A/B measurements of build variants; scripts/build_variant.py)
    v = os.environ.get("TM_LIB_VARIANT")
    return os.path.join(_HERE, f"libtm_{v}.so") if v else _LIB_PATH


def lib():
    """Load libtm.so; raise loudly if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        path = lib_path()
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(there is no CPU fallback for the CUDA path)")
        L = ctypes.CDLL(path)
        L.tm_plan_create.restype = ctypes.c_int
        L.tm_plan_create.argtypes = [ctypes.POINTER(_p), _i64, _i64, _i64, _u64, ctypes.c_int, _u32]
        L.tm_plan_query.restype = ctypes.c_int
        L.tm_plan_query.argtypes = [_p, ctypes.POINTER(PlanInfo)]
        L.tm_workspace_bytes.restype = ctypes.c_size_t
        L.tm_workspace_bytes.argtypes = [_p, _i64]
        L.tm_plan_destroy.restype = None
        L.tm_plan_destroy.argtypes = [_p]
        L.tm_generate.restype = ctypes.c_int
        L.tm_generate.argtypes = [_p, _i64, _i64, _d, _i64, _i64, _p, _i64, _p, _p, _p]
        L.tm_fold.restype = ctypes.c_int
        L.tm_fold.argtypes = [_p, _p, _i64, _i64, _i64, _i64, _p, _p, ctypes.c_int, _p, _p]
        L.tm_fold_template.restype = ctypes.c_int
        L.tm_fold_template.argtypes = [_p, _p, _i64, _p, _p]
        L.tm_correlate.restype = ctypes.c_int
        L.tm_correlate.argtypes = [_p, _p, _p, _p, _i64, _p, _p, _p, _p]
        L.tm_match.restype = ctypes.c_int
        L.tm_match.argtypes = [_p, _p, _p, _i64, _p, _p, _p]
        L.tm_run.restype = ctypes.c_int
        L.tm_run.argtypes = [_p, _p, _i64, _p, _i64, _p, _p, _p, _p]
        L.tm_correlate_match.restype = ctypes.c_int
        L.tm_correlate_match.argtypes = [_p, _p, _p, _p, _i64, _p, _p, _p, _p]
        L.tm_correlate_many.restype = ctypes.c_int
        L.tm_correlate_many.argtypes = [_p, _p, _p, _p, _i64, _p, _p, _p, _p]
        L.tm_run_host.restype = ctypes.c_int
        L.tm_run_host.argtypes = [_p, _p, _i64, _p, _i64, _i64, _p, _p, _p, _p, _p, _p, _p]
        L.tm_launch_count.restype = _u64
        L.tm_launch_count.argtypes = []
        L.tm_profile_events.restype = ctypes.c_int
        L.tm_profile_events.argtypes = [ctypes.POINTER(_p), ctypes.c_int]
        L.tm_run_path.restype = ctypes.c_int
        L.tm_run_path.argtypes = [_p, _i64]
        L.tm_correlate_match_part.restype = ctypes.c_int
        L.tm_correlate_match_part.argtypes = [_p, _p, _p, _p, _i64, ctypes.c_int, ctypes.c_int, _p, _p, _p]
        L.tm_match_keys.restype = ctypes.c_int
        L.tm_match_keys.argtypes = [_p, _p, _i64, _p, _p, _p]
        L.tm_mplan_create.restype = ctypes.c_int
        L.tm_mplan_create.argtypes = [ctypes.POINTER(_p), _i64, _i64, _p, ctypes.c_int, _u64, ctypes.c_int, _u32]
        L.tm_mplan_workspace_bytes.restype = ctypes.c_size_t
        L.tm_mplan_workspace_bytes.argtypes = [_p, _i64]
        L.tm_mplan_run.restype = ctypes.c_int
        L.tm_mplan_run.argtypes = [_p, _p, _i64, _p, _i64, _p, _p, _p, _p]
        L.tm_crt_multi.restype = ctypes.c_int
        L.tm_crt_multi.argtypes = [_p, _i64, ctypes.c_int, _p, _i64, _p, _p]
        L.tm_mplan_destroy.restype = None
        L.tm_mplan_destroy.argtypes = [_p]
        L.tm_run_fold_rows.restype = ctypes.c_int
        L.tm_run_fold_rows.argtypes = [_p, _i64, ctypes.POINTER(_i64)]
        L.tm_fold_reduce.restype = ctypes.c_int
        L.tm_fold_reduce.argtypes = [_p, _p, _i64, _i64, _i64, _i64, ctypes.c_int, _p, _p, ctypes.c_int, _p, _p]
        L.tm_probe_read_pattern.restype = ctypes.c_int
        L.tm_probe_read_pattern.argtypes = [_p, _i64, ctypes.c_int, _i64, _i64, ctypes.c_int, ctypes.c_int, _p]
        L.tm_probe_read_bw.restype = ctypes.c_int
        L.tm_probe_read_bw.argtypes = [_p, _i64, _p]
        L.tm_status_string.restype = ctypes.c_char_p
        L.tm_status_string.argtypes = [ctypes.c_int]
        L.tm_last_error.restype = ctypes.c_char_p
        L.tm_last_error.argtypes = []
        _lib = L
    return _lib


def launch_count() -> int:
    """Kernels launched by libtm in this process (tm_launch_count)."""
    return int(lib().tm_launch_count())


def profile_events(events):
    """tm_profile_events: list of 5 torch.cuda.Event (enable_timing) or None."""
    if events is None:
        _check(lib().tm_profile_events(None, 0), "tm_profile_events")
        return None
    arr = (_p * len(events))(*[e.cuda_event for e in events])
    _check(lib().tm_profile_events(arr, len(events)), "tm_profile_events")
    return arr  # keep alive while in use


def probe_read_bw(buf, stream=None):
    """tm_probe_read_bw: one read-only streaming pass over a device tensor (bench.py's
    live read-only ceiling; instrumentation, not part of the method)."""
    _check(lib().tm_probe_read_bw(_ptr(buf), buf.numel() * buf.element_size(), _stream(stream)), "tm_probe_read_bw")


def _check(rc: int, where: str):
    if rc != TM_OK:
        raise TMError(rc, where)


def _stream(stream):
    import torch
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _ptr(t):
    return None if t is None else t.data_ptr()


# test hook (TM_WS_POISON=1): every workspace the binding allocates starts as 0x7F bytes,
# so a kernel reading workspace memory it has not written shows up in the parity tests
# (TM_WS_POISON=0xFF etc. picks the byte)
_POISON = bool(os.environ.get("TM_WS_POISON"))
_POISON_BYTE = (int(os.environ.get("TM_WS_POISON") or "0", 0) & 0xFF) if _POISON else 0
if _POISON and _POISON_BYTE <= 1:
    _POISON_BYTE = 0x7F


def _poisoned(buf):
    if _POISON:
        buf.fill_(_POISON_BYTE)
    return buf


def _scratch(nbytes: int, device, stream):
    """A temporary device buffer used by a launch on `stream`: allocated while
    `stream` is current and recorded on it, so the caching allocator does not hand
    it to other work before the launch has finished with it."""
    import torch
    if stream is None or isinstance(stream, int):
        st = torch.cuda.current_stream(device) if stream is None else torch.cuda.ExternalStream(stream, device=device)
    else:
        st = stream
    with torch.cuda.stream(st):
        buf = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)
        if _POISON:
            buf.fill_(_POISON_BYTE)
    buf.record_stream(st)
    return buf


def _ld(x):
    """Row stride of a [batch][n] tensor (a single row may carry any stride in torch)."""
    return x.stride(0) if x.shape[0] > 1 else x.shape[1]


class Plan:
    """tm_plan: Alg. 1 step 2 (M1 = M or K, M2 = M1 + 1).  dtype is "int8" or "float32".
    engine (int8 only): None/"auto" (tensor cores when eligible), "ntt" or "tc".
    block: strategy 2 (Theorem 2's Block Phi, TM_BLOCK) instead of strategy 1."""

    def __init__(self, N: int, K: int, M: int = 0, seed: int = 0, dtype: str = "int8", binary: bool = True,
                 engine: str | None = None, alias_repair: bool = False, block: bool = False,
                 inputs_stable: bool = False, keep_y: bool = False):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1509_04863_b200.Plan needs a CUDA device (no CPU fallback)")
        self.dtype = {"int8": TM_I8, "float32": TM_F32}[str(dtype).replace("torch.", "")]
        flags = TM_BINARY if (binary and self.dtype == TM_I8) else 0
        if self.dtype == TM_I8:
            flags |= _ENGINES[engine]
        if alias_repair:
            flags |= TM_ALIAS_REPAIR
        if block:
            flags |= TM_BLOCK
        if inputs_stable:   # caller's x / t are not written while calls run (see tm.h)
            flags |= TM_INPUTS_STABLE
        if keep_y:          # test hook: the fused kernel keeps its y rows in ws
            flags |= TM_KEEP_Y
        h = _p()
        _check(lib().tm_plan_create(ctypes.byref(h), N, K, M, seed, self.dtype, flags), "tm_plan_create")
        self._h = h
        info = PlanInfo()
        _check(lib().tm_plan_query(h, ctypes.byref(info)), "tm_plan_query")
        self.info = info
        for f, _ in PlanInfo._fields_:
            setattr(self, f, getattr(info, f))
        self.x_dtype = torch.int8 if self.dtype == TM_I8 else torch.float32
        self.y_dtype = torch.int32 if self.dtype == TM_I8 else torch.float32
        self.r_dtype = torch.int64 if self.dtype == TM_I8 else torch.float32

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.tm_plan_destroy(h)
            self._h = None

    # ---- buffers (torch owns device memory) -------------------------------------
    def workspace(self, batch: int, device="cuda"):
        import torch
        n = lib().tm_workspace_bytes(self._h, batch)
        return _poisoned(torch.empty(max(int(n), 1), dtype=torch.uint8, device=device))

    def _tmp_ws(self, batch: int, device, stream):
        return _scratch(lib().tm_workspace_bytes(self._h, batch), device, stream)

    def fold_rows(self, ws, batch: int):
        """Views of the y1 / y2 rows tm_run writes into `ws` (tm_run_fold_rows; with
        keep_y=True the fused kernel keeps them): (y1 [batch][len_y1], y2 [batch][len_y2])."""
        import torch
        out = (_i64 * 4)()
        _check(lib().tm_run_fold_rows(self._h, batch, out), "tm_run_fold_rows")
        o1, ld1, o2, ld2 = (int(v) for v in out)
        es = 4
        y1 = ws[o1:o1 + batch * ld1 * es].view(self.y_dtype).view(batch, ld1)[:, :self.len_y1]
        y2 = ws[o2:o2 + batch * ld2 * es].view(self.y_dtype).view(batch, ld2)[:, :self.len_y2]
        return y1, y2

    # ---- entry points --------------------------------------------------------------
    def generate(self, pair0: int, batch: int, noise: float, offset: int = 0, length: int | None = None,
                 x=None, t=None, k0=None, want_x=True, stream=None, device="cuda"):
        import torch
        length = self.N - offset if length is None else length
        if want_x and x is None:
            x = torch.empty((batch, length), dtype=self.x_dtype, device=device)
        if t is None:
            t = torch.empty((batch, self.K), dtype=self.x_dtype, device=device)
        if k0 is None:
            k0 = torch.empty(batch, dtype=torch.int64, device=device)
        ldx = _ld(x) if x is not None and x.dim() == 2 else length
        _check(lib().tm_generate(self._h, pair0, batch, float(noise), offset, length, _ptr(x), ldx, _ptr(t),
                                 _ptr(k0), _stream(stream)), "tm_generate")
        return x, t, k0

    def fold(self, x, offset: int = 0, length: int | None = None, y1=None, y2=None, accumulate=False,
             ws=None, stream=None):
        import torch
        batch = x.shape[0]
        length = x.shape[1] if length is None else length
        if y1 is None:
            y1 = torch.zeros((batch, self.len_y1), dtype=self.y_dtype, device=x.device)
        if y2 is None:
            y2 = torch.zeros((batch, self.len_y2), dtype=self.y_dtype, device=x.device)
        if ws is None:
            ws = self._tmp_ws(batch, x.device, stream)
        _check(lib().tm_fold(self._h, _ptr(x), _ld(x), batch, offset, length, _ptr(y1), _ptr(y2),
                             int(accumulate), _ptr(ws), _stream(stream)), "tm_fold")
        return y1, y2

    def fold_reduce(self, x, dst_y1, dst_y2, offset: int = 0, length: int | None = None, multicast: bool = False,
                    ws=None, stream=None):
        """tm_fold_reduce: ADD this chunk's fold into every destination (lists of
        device pointers (ints) or tensors: peer-mapped buffers, or one multicast
        address each with multicast=True)."""
        batch = x.shape[0]
        length = x.shape[1] if length is None else length
        d1 = [v if isinstance(v, int) else v.data_ptr() for v in dst_y1]
        d2 = [v if isinstance(v, int) else v.data_ptr() for v in dst_y2]
        if len(d1) != len(d2):
            raise ValueError("dst_y1 and dst_y2 need the same length")
        a1 = (_p * len(d1))(*d1)
        a2 = (_p * len(d2))(*d2)
        if ws is None:
            ws = self._tmp_ws(batch, x.device, stream)
        _check(lib().tm_fold_reduce(self._h, _ptr(x), _ld(x), batch, offset, length, len(d1), a1, a2, int(multicast),
                                    _ptr(ws), _stream(stream)), "tm_fold_reduce")

    def fold_template(self, t, tf=None, stream=None):
        import torch
        batch = t.shape[0]
        if tf is None:
            tf = torch.empty((batch, self.tf_bytes), dtype=torch.uint8, device=t.device)
        _check(lib().tm_fold_template(self._h, _ptr(t), batch, _ptr(tf), _stream(stream)), "tm_fold_template")
        return tf

    def correlate(self, y1, y2, tf, r1=None, r2=None, ws=None, stream=None):
        import torch
        batch = y1.shape[0]
        if r1 is None:
            r1 = torch.empty((batch, self.M1), dtype=self.r_dtype, device=y1.device)
        if r2 is None:
            r2 = torch.empty((batch, self.M2), dtype=self.r_dtype, device=y1.device)
        if ws is None:
            ws = self._tmp_ws(batch, y1.device, stream)
        _check(lib().tm_correlate(self._h, _ptr(y1), _ptr(y2), _ptr(tf), batch, _ptr(r1), _ptr(r2), _ptr(ws),
                                  _stream(stream)), "tm_correlate")
        return r1, r2

    def match(self, r1, r2, residues=None, k=None, stream=None):
        import torch
        batch = r1.shape[0]
        if residues is None:
            residues = torch.empty((batch, 2), dtype=torch.int32, device=r1.device)
        if k is None:
            k = torch.empty(batch, dtype=torch.int64, device=r1.device)
        _check(lib().tm_match(self._h, _ptr(r1), _ptr(r2), batch, _ptr(residues), _ptr(k), _stream(stream)),
               "tm_match")
        return residues, k

    def run(self, x, t, residues=None, k=None, ws=None, stream=None):
        import torch
        batch = x.shape[0]
        if residues is None:
            residues = torch.empty((batch, 2), dtype=torch.int32, device=x.device)
        if k is None:
            k = torch.empty(batch, dtype=torch.int64, device=x.device)
        if ws is None:
            ws = self._tmp_ws(batch, x.device, stream)
        _check(lib().tm_run(self._h, _ptr(x), _ld(x), _ptr(t), batch, _ptr(residues), _ptr(k), _ptr(ws),
                            _stream(stream)), "tm_run")
        return residues, k

    def correlate_match(self, y1, y2, t, residues=None, k=None, ws=None, stream=None):
        """tm_correlate_match: steps 4-9 on already-folded (e.g. all-reduced) y1, y2."""
        import torch
        batch = y1.shape[0]
        if residues is None:
            residues = torch.empty((batch, 2), dtype=torch.int32, device=y1.device)
        if k is None:
            k = torch.empty(batch, dtype=torch.int64, device=y1.device)
        if ws is None:
            ws = self._tmp_ws(batch, y1.device, stream)
        _check(lib().tm_correlate_match(self._h, _ptr(y1), _ptr(y2), _ptr(t), batch, _ptr(residues), _ptr(k),
                                        _ptr(ws), _stream(stream)), "tm_correlate_match")
        return residues, k

    def correlate_match_part(self, y1, y2, t, part: int, nparts: int, keys=None, ws=None, stream=None):
        """tm_correlate_match_part: this part's best (r, k) per modulus as int64 keys [batch][2]."""
        import torch
        batch = y1.shape[0]
        if keys is None:
            keys = torch.empty((batch, 2), dtype=torch.int64, device=y1.device)
        if ws is None:
            ws = self._tmp_ws(batch, y1.device, stream)
        _check(lib().tm_correlate_match_part(self._h, _ptr(y1), _ptr(y2), _ptr(t), batch, part, nparts, _ptr(keys),
                                             _ptr(ws), _stream(stream)), "tm_correlate_match_part")
        return keys

    def match_keys(self, keys, residues=None, k=None, stream=None):
        """tm_match_keys: (MAX-reduced) keys -> residues, k (steps 8-9)."""
        import torch
        batch = keys.shape[0]
        if residues is None:
            residues = torch.empty((batch, 2), dtype=torch.int32, device=keys.device)
        if k is None:
            k = torch.empty(batch, dtype=torch.int64, device=keys.device)
        _check(lib().tm_match_keys(self._h, _ptr(keys), batch, _ptr(residues), _ptr(k), _stream(stream)),
               "tm_match_keys")
        return residues, k

    def run_path(self, batch: int) -> int:
        """tm_run_path: which kernel sequence tm_run launches for this batch (instrumentation)."""
        return int(lib().tm_run_path(self._h, batch))

    def correlate_many(self, y1, y2, t, residues=None, k=None, ws=None, stream=None):
        """tm_correlate_many: one folded signal (y1 [len_y1], y2 [len_y2]) against
        templates t [n][K] -> residues [n][2], k [n]."""
        import torch
        n = t.shape[0]
        if residues is None:
            residues = torch.empty((n, 2), dtype=torch.int32, device=t.device)
        if k is None:
            k = torch.empty(n, dtype=torch.int64, device=t.device)
        if ws is None:
            ws = self._tmp_ws(n, t.device, stream)
        _check(lib().tm_correlate_many(self._h, _ptr(y1), _ptr(y2), _ptr(t), n, _ptr(residues), _ptr(k), _ptr(ws),
                                       _stream(stream)), "tm_correlate_many")
        return residues, k

    def run_host(self, x_host, t_host, chunk: int, residues_host, k_host, dev_x, dev_t, dev_out, ws, stream=None):
        """tm_run_host: x_host/t_host/residues_host/k_host are (pinned) CPU tensors."""
        batch = x_host.shape[0]
        _check(lib().tm_run_host(self._h, _ptr(x_host), _ld(x_host), _ptr(t_host), batch, chunk,
                                 _ptr(residues_host), _ptr(k_host), _ptr(dev_x), _ptr(dev_t), _ptr(dev_out),
                                 _ptr(ws), _stream(stream)), "tm_run_host")

    def run_host_buffers(self, batch: int, chunk: int, device="cuda"):
        """Device staging buffers for run_host (double-buffered chunks)."""
        import torch
        dev_x = torch.empty((2 * chunk, self.N), dtype=self.x_dtype, device=device)
        dev_t = torch.empty((2 * chunk, self.K), dtype=self.x_dtype, device=device)
        dev_out = torch.empty(((batch * 8 + 255) // 256 * 256) + batch * 8, dtype=torch.uint8, device=device)
        return dev_x, dev_t, dev_out, self.workspace(chunk, device)


class MultiPlan:
    """tm_mplan: Theorem 4 with alpha pairwise co-prime moduli.
    moduli: alpha integers, K <= M_j < 2^31, product > N."""

    def __init__(self, N: int, K: int, moduli, seed: int = 0, dtype: str = "int8", binary: bool = True,
                 engine: str | None = None, block: bool = False):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1509_04863_b200.MultiPlan needs a CUDA device (no CPU fallback)")
        self.N, self.K = N, K
        self.moduli = [int(m) for m in moduli]
        self.alpha = len(self.moduli)
        dt = {"int8": TM_I8, "float32": TM_F32}[str(dtype).replace("torch.", "")]
        flags = TM_BINARY if (binary and dt == TM_I8) else 0
        if dt == TM_I8:
            flags |= _ENGINES[engine]
        if block:
            flags |= TM_BLOCK
        self._M = (ctypes.c_int64 * self.alpha)(*self.moduli)
        h = _p()
        _check(lib().tm_mplan_create(ctypes.byref(h), N, K, ctypes.cast(self._M, _p), self.alpha, seed, dt, flags),
               "tm_mplan_create")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.tm_mplan_destroy(h)
            self._h = None

    def workspace(self, batch: int, device="cuda"):
        import torch
        n = lib().tm_mplan_workspace_bytes(self._h, batch)
        return _poisoned(torch.empty(max(int(n), 1), dtype=torch.uint8, device=device))

    def run(self, x, t, residues=None, k=None, ws=None, stream=None):
        """Steps 3-7 per modulus, then Garner's CRT: (residues [batch][alpha], k [batch])."""
        import torch
        batch = x.shape[0]
        if residues is None:
            residues = torch.empty((batch, self.alpha), dtype=torch.int32, device=x.device)
        if k is None:
            k = torch.empty(batch, dtype=torch.int64, device=x.device)
        if ws is None:
            ws = _scratch(lib().tm_mplan_workspace_bytes(self._h, batch), x.device, stream)
        _check(lib().tm_mplan_run(self._h, _ptr(x), _ld(x), _ptr(t), batch, _ptr(residues), _ptr(k), _ptr(ws),
                                  _stream(stream)), "tm_mplan_run")
        return residues, k


def crt_multi(residues, moduli, N: int, k=None, stream=None):
    """tm_crt_multi: steps 8-9 alone for residues int32 [batch][alpha] (device)."""
    import torch
    batch, alpha = residues.shape
    if k is None:
        k = torch.empty(batch, dtype=torch.int64, device=residues.device)
    M = (ctypes.c_int64 * alpha)(*[int(m) for m in moduli])
    _check(lib().tm_crt_multi(_ptr(residues), batch, alpha, ctypes.cast(M, _p), N, _ptr(k), _stream(stream)),
           "tm_crt_multi")
    return k
