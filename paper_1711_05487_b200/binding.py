"""ctypes binding of include/spmv.h (same names as the C ABI, minus the prefix).

Accepts numpy arrays (host) or torch tensors (host or CUDA) and passes their
raw pointers; the library detects host vs device memory itself.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_PATH = os.environ.get("SPMV_LIB_PATH") or os.path.join(_HERE, "libspmv.so")  # override: experiment builds
if not os.path.exists(_PATH):
    raise ImportError(f"{_PATH} is missing: build it with `make spmv` or __graft_entry__.build() "
                      "(there is no CPU fallback)")
lib = ctypes.CDLL(_PATH)

VARIANTS = {"auto": 0, "vector": 1, "stream": 2, "merge": 3, "split": 4, "nnzsplit": 5}
VARIANT_NAMES = {v: k for k, v in VARIANTS.items()}
CLASSES = {"MB": 1, "ML": 2, "IMB": 4, "CMP": 8}
ARR = {"tile_rows": 1, "merge_rows": 2, "merge_nnz": 3, "chunk_row": 4, "chunk_begin": 5, "chunk_end": 6,
       "dcol": 7, "head": 8, "anchor": 9, "decoded": 10, "shard_bounds": 11, "nz_rowmap": 12, "nz_rpc": 13,
       "nz_tile_q": 14, "nz_hot_cols": 15, "d8_codes": 16, "d8_rlen": 17, "d8_dict": 18, "pat_ids": 19,
       "pat_len": 20, "pat_ofs": 21}
_ARR_DTYPE = {1: np.int64, 2: np.int64, 3: np.int64, 4: np.int64, 5: np.int64, 6: np.int64, 7: np.uint16,
              8: np.int32, 9: np.int32, 10: np.int32, 11: np.int64, 12: np.int64, 13: np.int64, 14: np.int64,
              15: np.int64, 16: np.uint8, 17: np.uint8, 18: np.int64, 19: np.uint8, 20: np.int64, 21: np.int64}


class Options(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_int32), ("force_variant", ctypes.c_int32), ("force_vs", ctypes.c_int32),
                ("d16", ctypes.c_int32), ("xwin", ctypes.c_int32), ("validate", ctypes.c_int32),
                ("l_split", ctypes.c_int64), ("k_long", ctypes.c_int64), ("tile_nnz", ctypes.c_int64),
                ("merge_items", ctypes.c_int64), ("long_chunk", ctypes.c_int64),
                ("emulate_devices", ctypes.c_int32), ("stages", ctypes.c_int32), ("seg", ctypes.c_int32),
                ("long_mode", ctypes.c_int32), ("split_bins", ctypes.c_int32), ("hot_x", ctypes.c_int32),
                ("select_mode", ctypes.c_int32), ("reserved", ctypes.c_int32 * 1),
                ("t_imb", ctypes.c_double), ("t_ml", ctypes.c_double), ("approx_tol", ctypes.c_double),
                ("force_classes", ctypes.c_int32), ("pad_", ctypes.c_int32)]

    @classmethod
    def _names(cls):
        return {f[0] for f in cls._fields_} - {"struct_size", "reserved", "pad_"}

    @classmethod
    def make(cls, **kw):
        o = cls()
        lib.spmv_options_default(ctypes.byref(o))
        for k, v in kw.items():
            if k == "no_aligned":  # reserved[0]: disable row-aligned STREAM tiles
                o.reserved[0] = int(v)
                continue
            if k == "force_variant" and isinstance(v, str):
                v = VARIANTS[v]
            if k not in cls._names():
                raise TypeError(f"unknown spmv option {k!r}")
            setattr(o, k, v)
        return o


class Features(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int64) for k in
                ("n", "nnz", "nnz_min", "nnz_max", "n_empty", "n_long", "nnz_long", "n_short", "max_short")] + \
               [(k, ctypes.c_uint64) for k in ("s1", "s2", "s1_short", "s2_short")] + \
               [(k, ctypes.c_int64) for k in ("maxgap", "misses")] + \
               [(k, ctypes.c_double) for k in ("nnz_avg", "nnz_sd", "avg_short", "sd_short")] + \
               [("n_cols", ctypes.c_int64), ("n_big_gaps", ctypes.c_int64), ("col_min", ctypes.c_int64),
                ("col_max", ctypes.c_int64), ("n_deltas", ctypes.c_int64)]


class DeviceProps(ctypes.Structure):
    _fields_ = [("sm_count", ctypes.c_int32), ("cc_major", ctypes.c_int32), ("cc_minor", ctypes.c_int32),
                ("pad_", ctypes.c_int32), ("l2_bytes", ctypes.c_int64), ("persisting_l2_max", ctypes.c_int64),
                ("access_window_max", ctypes.c_int64), ("global_mem_bytes", ctypes.c_int64)]


class Selection(ctypes.Structure):
    _fields_ = [("variant", ctypes.c_int32), ("vs", ctypes.c_int32), ("d16", ctypes.c_int32),
                ("xwin", ctypes.c_int32), ("classes", ctypes.c_int32), ("seg", ctypes.c_int32)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("n_rows", ctypes.c_int64), ("n_cols", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("rowptr_bytes", ctypes.c_int32), ("ngpus", ctypes.c_int32), ("sel", Selection),
                ("feat", Features), ("d16_width", ctypes.c_int32), ("d16_n_esc", ctypes.c_int32),
                ("tile_nnz", ctypes.c_int64), ("n_tiles", ctypes.c_int64), ("merge_items", ctypes.c_int64),
                ("n_merge_tiles", ctypes.c_int64), ("l_split", ctypes.c_int64), ("long_chunk", ctypes.c_int64),
                ("n_long_chunks", ctypes.c_int64), ("upload_ms", ctypes.c_double), ("inspect_ms", ctypes.c_double),
                ("select_ms", ctypes.c_double), ("encode_ms", ctypes.c_double), ("device_bytes", ctypes.c_int64),
                ("shard_bounds", ctypes.c_int64 * 9), ("tile_stride", ctypes.c_int64),
                ("tiles_row_aligned", ctypes.c_int32), ("rows_per_tile", ctypes.c_int32), ("n_nz_rows", ctypes.c_int64),
                ("n_nz_tiles", ctypes.c_int64), ("n_hot", ctypes.c_int64), ("hot_cover", ctypes.c_double)] + \
               [(k, ctypes.c_double) for k in ("p_csr", "p_mb", "p_ml", "p_imb", "p_cmp", "p_peak", "bmax")] + \
               [("profile_vs", ctypes.c_int32), ("profile_ctas", ctypes.c_int32), ("profile_ms", ctypes.c_double),
               ("x_reuse", ctypes.c_double), ("nz_gather_l2", ctypes.c_int32), ("stream_stages", ctypes.c_int32),
               ("d8_n_dict", ctypes.c_int32), ("stream_grid", ctypes.c_int32), ("kernel_bytes", ctypes.c_int64),
               ("long_mode", ctypes.c_int32), ("long_rg", ctypes.c_int32), ("iter_push", ctypes.c_int32),
               ("long_c16", ctypes.c_int32), ("p_stream", ctypes.c_double),
               ("d8_patterns", ctypes.c_int32), ("pad3_", ctypes.c_int32)]


_vp, _i64, _i32, _d = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
lib.spmv_options_default.argtypes = [ctypes.POINTER(Options)]
lib.spmv_plan_create.argtypes = [_i64, _i64, _vp, _vp, _vp, ctypes.c_int]
lib.spmv_plan_create.restype = _vp
lib.spmv_plan_create_ex.argtypes = [ctypes.POINTER(_vp), _i64, _i64, _i64, _vp, ctypes.c_int, _vp, _vp, ctypes.c_int,
                                    ctypes.POINTER(Options)]
lib.spmv_plan_destroy.argtypes = [_vp]
lib.spmv_plan_update_values.argtypes = [_vp, _vp]
lib.spmv_abi_sizes.argtypes = [ctypes.POINTER(_i64), ctypes.c_int]
lib.spmv_execute.argtypes = [_vp, _vp, _vp]
lib.spmv_execute_async.argtypes = [_vp, _vp, _vp]
lib.spmv_execute_stage.argtypes = [_vp, _vp, _vp, ctypes.c_int]
lib.spmv_iterate.argtypes = [_vp, _vp, _vp, ctypes.c_int, ctypes.POINTER(_d), _vp]
lib.spmv_norm_partial_count.restype = _i32
lib.spmv_norm_partials.argtypes = [_vp, _vp, _vp]
lib.spmv_normalize.argtypes = [_vp, _vp, _vp, ctypes.c_int, _vp, _vp]
lib.spmv_norm_step.argtypes = [_vp, _vp, ctypes.c_int, _vp, _vp]
if hasattr(lib, "spmv_iter_step"):  # (experiment builds of older sources lack it)
    lib.spmv_iter_step.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp]
lib.spmv_execute_norm.argtypes = [_vp, _vp, _vp, _vp]
lib.spmv_unit.argtypes = [_vp, _vp, ctypes.c_int64, _vp, _vp]
lib.spmv_plan_query.argtypes = [_vp, ctypes.POINTER(PlanInfo)]
IPC_HANDLE_BYTES = 64  # SPMV_IPC_HANDLE_BYTES
lib.spmv_plan_replicas.argtypes = [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp)]
lib.spmv_iter_push_capable.argtypes = [_vp]
lib.spmv_ipc_export.argtypes = [_vp, _vp, _vp]
lib.spmv_ipc_open.argtypes = [_vp, _vp, ctypes.POINTER(_vp)]
lib.spmv_iter_step_push.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _i64]


class Table1(ctypes.Structure):
    _fields_ = [("size_fits_l2", ctypes.c_int32), ("pad_", ctypes.c_int32)] + \
               [(k, ctypes.c_double) for k in ("density", "nnz_min", "nnz_max", "nnz_avg", "nnz_sd", "bw_min",
                                               "bw_max", "bw_avg", "bw_sd", "scatter_avg", "scatter_sd",
                                               "clustering_avg", "misses_avg")] + [("n_nonempty", ctypes.c_int64)]


lib.spmv_plan_table1.argtypes = [_vp, ctypes.POINTER(Table1)]
lib.spmv_plan_x_device.argtypes = [_vp, ctypes.c_int]
lib.spmv_plan_x_device.restype = _vp
lib.spmv_plan_y_device.argtypes = [_vp, ctypes.c_int]
lib.spmv_plan_y_device.restype = _vp
lib.spmv_plan_stream.argtypes = [_vp, ctypes.c_int]
lib.spmv_plan_stream.restype = _vp
lib.spmv_plan_export.argtypes = [_vp, ctypes.c_int, ctypes.c_int, _vp]
lib.spmv_plan_export.restype = _i64
lib.spmv_shard_bounds.argtypes = [_i64, _vp, ctypes.c_int, ctypes.c_int, _vp]
lib.spmv_select.argtypes = [ctypes.POINTER(Features), ctypes.POINTER(DeviceProps), ctypes.c_int,
                            ctypes.POINTER(Options), ctypes.POINTER(Selection)]
lib.spmv_device_query.argtypes = [ctypes.c_int, ctypes.POINTER(DeviceProps)]
lib.spmv_last_error.restype = ctypes.c_char_p
lib.spmv_kernel_launches.restype = _i64


class SpmvError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"spmv status {status}: {msg}")
        self.status = status
        self.msg = msg


def _check(rc):
    if rc != 0:
        raise SpmvError(int(rc), lib.spmv_last_error().decode())
    return rc


def _ptr(a):
    """Raw pointer of a numpy array or torch tensor (contiguity is the caller's job)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"], "array must be contiguous"
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        assert a.is_contiguous(), "tensor must be contiguous"
        return a.data_ptr()
    if isinstance(a, int):
        return a
    raise TypeError(type(a))


def _elem_bytes(a):
    if isinstance(a, np.ndarray):
        return a.dtype.itemsize
    return a.element_size()


def _numel(a):
    return a.size if isinstance(a, np.ndarray) else a.numel()


def kernel_launches() -> int:
    return int(lib.spmv_kernel_launches())


def norm_partial_count() -> int:
    return int(lib.spmv_norm_partial_count())


def shard_bounds(rowptr: np.ndarray, G: int) -> np.ndarray:
    rp = np.ascontiguousarray(rowptr)
    out = np.empty(G + 1, np.int64)
    _check(lib.spmv_shard_bounds(rp.size - 1, rp.ctypes.data, rp.dtype.itemsize, G, out.ctypes.data))
    return out


def select(features: dict, props: dict, rowptr_bytes: int, **opts) -> dict:
    f = Features(**{k: features[k] for k, _ in Features._fields_})
    d = DeviceProps(**{k: props.get(k, 0) for k, _ in DeviceProps._fields_})
    o = Options.make(**opts)
    s = Selection()
    _check(lib.spmv_select(ctypes.byref(f), ctypes.byref(d), rowptr_bytes, ctypes.byref(o), ctypes.byref(s)))
    return {k: getattr(s, k) for k, _ in Selection._fields_ if k != "pad_"}


def device_query(dev: int = 0) -> dict:
    d = DeviceProps()
    _check(lib.spmv_device_query(dev, ctypes.byref(d)))
    return {k: getattr(d, k) for k, _ in DeviceProps._fields_ if k != "pad_"}


class Plan:
    """spmv_plan_create_ex + execute/iterate/query/export/destroy."""

    def __init__(self, rowptr, colind, values, n_cols=None, ngpus=1, **opts):
        n_rows = _numel(rowptr) - 1
        nnz = _numel(colind)
        self._h = _vp()
        self.options = Options.make(**opts)
        # keep references alive for the duration of the (synchronous) create
        self._keep = (rowptr, colind, values)
        _check(lib.spmv_plan_create_ex(ctypes.byref(self._h), n_rows, n_rows if n_cols is None else n_cols, nnz,
                                       _ptr(rowptr), _elem_bytes(rowptr), _ptr(colind), _ptr(values), ngpus,
                                       ctypes.byref(self.options)))
        self._keep = None
        self.n_rows = n_rows
        self.n_cols = n_rows if n_cols is None else n_cols
        self.nnz = nnz

    @property
    def handle(self):
        return self._h.value

    def destroy(self):
        if self._h and self._h.value:
            lib.spmv_plan_destroy(self._h)
            self._h = _vp()

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    def update_values(self, values):
        """spmv_plan_update_values: same pattern, new values (CSR order, host or device)."""
        if _numel(values) != self.nnz:
            raise ValueError(f"values must have nnz = {self.nnz} entries")
        _check(lib.spmv_plan_update_values(self._h, _ptr(values)))

    def execute(self, x, y=None):
        if y is None:
            y = np.empty(self.n_rows, np.float64)
        _check(lib.spmv_execute(self._h, _ptr(x), _ptr(y)))
        return y

    def execute_async(self, x, y):
        _check(lib.spmv_execute_async(self._h, _ptr(x), _ptr(y)))

    def execute_stage(self, x, y, stage):
        _check(lib.spmv_execute_stage(self._h, _ptr(x), _ptr(y), int(stage)))

    def iterate(self, x0, iters, x_out=None):
        if x_out is None:
            x_out = np.empty(self.n_cols, np.float64)
        nu = np.zeros(iters, np.float64)
        last = ctypes.c_double(0.0)
        rc = lib.spmv_iterate(self._h, _ptr(x0), _ptr(x_out), int(iters), ctypes.byref(last), nu.ctypes.data)
        if rc != 0:
            raise SpmvError(int(rc), lib.spmv_last_error().decode())
        return x_out, nu

    def norm_partials(self, y, partials):
        _check(lib.spmv_norm_partials(self._h, _ptr(y), _ptr(partials)))

    def normalize(self, y, partials, count, x_out, nu_dev):
        _check(lib.spmv_normalize(self._h, _ptr(y), _ptr(partials), int(count), _ptr(x_out), _ptr(nu_dev)))

    def execute_norm(self, x, y, partials):
        _check(lib.spmv_execute_norm(self._h, _ptr(x), _ptr(y), _ptr(partials)))

    def norm_step(self, partials, count, nn, nu_k):
        _check(lib.spmv_norm_step(self._h, _ptr(partials), int(count), _ptr(nn), _ptr(nu_k)))

    def iter_step(self, x, y, partials, nn, nu_k=None):
        _check(lib.spmv_iter_step(self._h, _ptr(x), _ptr(y), _ptr(partials), _ptr(nn), _ptr(nu_k)))

    def iter_step_push(self, x, y, partials, nn, push_lo, push_lo_end, push_hi, push_hi_begin):
        _check(lib.spmv_iter_step_push(self._h, _ptr(x), _ptr(y), _ptr(partials), _ptr(nn), _ptr(push_lo),
                                       int(push_lo_end), _ptr(push_hi), int(push_hi_begin)))

    def replicas(self):
        """spmv_plan_replicas: device pointers (ints) of the plan's two x replicas."""
        a, b = _vp(), _vp()
        _check(lib.spmv_plan_replicas(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def push_capable(self) -> bool:
        return bool(lib.spmv_iter_push_capable(self._h))

    def ipc_export(self, replica) -> bytes:
        h = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
        _check(lib.spmv_ipc_export(self._h, _ptr(replica), h))
        return h.raw

    def ipc_open(self, handle: bytes) -> int:
        if len(handle) != IPC_HANDLE_BYTES:
            raise ValueError("IPC handle must be %d bytes" % IPC_HANDLE_BYTES)
        d = _vp()
        _check(lib.spmv_ipc_open(self._h, ctypes.create_string_buffer(bytes(handle), IPC_HANDLE_BYTES),
                                 ctypes.byref(d)))
        return d.value

    def unit(self, y, nn, x_out):
        _check(lib.spmv_unit(self._h, _ptr(y), int(_numel(y)), _ptr(nn), _ptr(x_out)))

    def info(self) -> dict:
        i = PlanInfo()
        _check(lib.spmv_plan_query(self._h, ctypes.byref(i)))
        d = {k: getattr(i, k) for k, _ in PlanInfo._fields_ if k not in ("sel", "feat", "pad_", "pad3_", "shard_bounds")}
        d["sel"] = {k: getattr(i.sel, k) for k, _ in Selection._fields_ if k != "pad_"}
        d["variant"] = VARIANT_NAMES[i.sel.variant]
        d["classes"] = [k for k, v in CLASSES.items() if i.sel.classes & v]
        d["feat"] = {k: getattr(i.feat, k) for k, _ in Features._fields_}
        d["shard_bounds"] = list(i.shard_bounds)[: i.ngpus + 1]
        return d

    def table1(self) -> dict:
        t = Table1()
        _check(lib.spmv_plan_table1(self._h, ctypes.byref(t)))
        return {k: getattr(t, k) for k, _ in Table1._fields_ if k != "pad_"}

    def export(self, which, g=0) -> np.ndarray:
        w = ARR[which] if isinstance(which, str) else which
        n = lib.spmv_plan_export(self._h, g, w, None)
        if n < 0:
            raise SpmvError(int(n), lib.spmv_last_error().decode())
        out = np.empty(n, _ARR_DTYPE[w])
        if n:
            rc = lib.spmv_plan_export(self._h, g, w, out.ctypes.data)
            if rc < 0:
                raise SpmvError(int(rc), lib.spmv_last_error().decode())
        return out

    def x_device(self, g=0) -> int:
        return lib.spmv_plan_x_device(self._h, g)

    def y_device(self, g=0) -> int:
        return lib.spmv_plan_y_device(self._h, g)

    def stream(self, g=0) -> int:
        return lib.spmv_plan_stream(self._h, g)
