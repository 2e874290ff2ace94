"""ctypes binding of librp (include/rp.h). Argument marshalling only.

Every C entry point has a same-named Python function here (``rp_init``,
``rp_preduce``, ...). They raise :class:`RPError` on a non-zero status, with
the library's thread-local message. :class:`Context` is a small convenience
wrapper over the same calls. Device pointers are passed as integers
(``tensor.data_ptr()``); streams as ``cudaStream_t`` integers
(``torch.cuda.Stream.cuda_stream``).
"""
import ctypes
import os

RP_OK = 0
RP_EINVAL = -1
RP_ESTATE = -2
RP_EPROTO = -3
RP_ECONFLICT = -4
RP_ETIMEOUT = -5
RP_ECUDA = -6
RP_ENOMEM = -7
RP_ENODEV = -8
RP_EAGAIN = -9

RP_MAX_WORLD = 64
RP_MAX_GROUP = 16
RP_FLAG_TRACE = 0x1
RP_FLAG_TIMING = 0x2
RP_FLAG_SHARED_GG = 0x4
RP_FLAG_RANDOM_GG = 0x8
RP_FLAG_INTER_INTRA = 0x10
RP_FLAG_EMULATE = 0x20
RP_FLAG_GRAPH = 0x40
RP_DTYPE_F32 = 0
RP_DTYPE_BF16 = 1
RP_SCHED_PAPER4 = 1
RP_SCHED_SHIFT_K = 2
RP_SCHED_GG = -1
RP_WAIT_DEVICE = -1

_HERE = os.path.dirname(os.path.abspath(__file__))


def library_path():
    return os.environ.get("RP_LIBRARY", os.path.join(_HERE, "librp.so"))


class rp_config(ctypes.Structure):
    _fields_ = [
        ("world", ctypes.c_int32),
        ("n_gpus", ctypes.c_int32),
        ("n_params", ctypes.c_int64),
        ("workers_per_gpu", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("group_size", ctypes.c_int32),
        ("c_thres", ctypes.c_int32),
        ("nodes", ctypes.c_int32),
        ("seed_gd", ctypes.c_uint64),
        ("flags", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("job_id", ctypes.c_uint64),
        ("watchdog_s", ctypes.c_int32),
        ("reserved", ctypes.c_int32 * 3),
    ]


class rp_group(ctypes.Structure):
    _fields_ = [
        ("seq", ctypes.c_int64),
        ("size", ctypes.c_int32),
        ("members", ctypes.c_int32 * RP_MAX_GROUP),
    ]

    def member_list(self):
        return [int(self.members[i]) for i in range(self.size)]

    @classmethod
    def make(cls, seq, members):
        g = cls()
        g.seq = seq
        g.size = len(members)
        for i in range(RP_MAX_GROUP):
            g.members[i] = members[i] if i < len(members) else -1
        return g

    def __repr__(self):
        return f"rp_group(seq={self.seq}, members={self.member_list()})"


class rp_stats(ctypes.Structure):
    _fields_ = [(name, ctypes.c_int64) for name in (
        "groups_launched", "singleton_groups", "cross_gpu_groups", "kernel_launches", "gd_calls",
        "gg_requests", "max_gb_depth", "lock_assertions", "bytes_hbm", "bytes_nvlink", "gg_pending",
        "gg_granted", "nvls_groups")]

    def as_dict(self):
        return {name: int(getattr(self, name)) for name, _ in self._fields_}


class rp_timing(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_int64), ("total_ms", ctypes.c_double), ("min_ms", ctypes.c_double),
                ("max_ms", ctypes.c_double), ("bytes_hbm", ctypes.c_int64), ("bytes_nvlink", ctypes.c_int64),
                ("local_launches", ctypes.c_int64), ("local_ms", ctypes.c_double),
                ("local_bytes_hbm", ctypes.c_int64), ("cross_launches", ctypes.c_int64),
                ("cross_ms", ctypes.c_double), ("cross_bytes_nvlink", ctypes.c_int64),
                ("cross_bytes_hbm", ctypes.c_int64)]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


RP_MAX_LOCAL = 16
RP_IPC_HANDLE_BYTES = 64


class rp_peer_info(ctypes.Structure):
    _fields_ = [
        ("rank", ctypes.c_int32),
        ("n_local", ctypes.c_int32),
        ("first_worker", ctypes.c_int32),
        ("pid", ctypes.c_int32),
        ("flags_handle", ctypes.c_uint8 * RP_IPC_HANDLE_BYTES),
        ("flags_offset", ctypes.c_int64),
        ("stage_handle", ctypes.c_uint8 * RP_IPC_HANDLE_BYTES),
        ("stage_offset", ctypes.c_int64),
        ("stage_region_bytes", ctypes.c_int64),
        ("x_handle", (ctypes.c_uint8 * RP_IPC_HANDLE_BYTES) * RP_MAX_LOCAL),
        ("x_offset", ctypes.c_int64 * RP_MAX_LOCAL),
    ]


class rp_launch_record(ctypes.Structure):
    _fields_ = [
        ("ms", ctypes.c_double),
        ("bytes_hbm", ctypes.c_int64),
        ("bytes_nvlink", ctypes.c_int64),
        ("batch", ctypes.c_int64),
        ("cross", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


class RPError(RuntimeError):
    def __init__(self, status, func, message):
        super().__init__(f"{func} failed: status {status}: {message}")
        self.status = status


_P = ctypes.c_void_p
_CTX = ctypes.c_void_p
# int (*rp_barrier_fn)(void* user, int32_t local_status)
RP_BARRIER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int32)
# name -> (restype, argtypes); the list is also what the ABI test checks against rp.h
_SIGNATURES = {
    "rp_init": (ctypes.c_int, [ctypes.POINTER(rp_config), ctypes.POINTER(_CTX)]),
    "rp_finalize": (ctypes.c_int, [_CTX]),
    "rp_bind_worker": (ctypes.c_int, [_CTX, ctypes.c_int32, _P, _P]),
    "rp_bind_worker_bf16": (ctypes.c_int, [_CTX, ctypes.c_int32, _P, _P]),
    "rp_worker_stream": (ctypes.c_int, [_CTX, ctypes.c_int32, ctypes.POINTER(_P)]),
    "rp_set_worker_stream": (ctypes.c_int, [_CTX, ctypes.c_int32, _P]),
    "rp_peer_export": (ctypes.c_int, [_CTX, ctypes.POINTER(rp_peer_info)]),
    "rp_peer_import": (ctypes.c_int, [_CTX, ctypes.POINTER(rp_peer_info), ctypes.c_int32]),
    "rp_nvls_supported": (ctypes.c_int, [_CTX, ctypes.POINTER(ctypes.c_int32)]),
    "rp_nvls_enable": (ctypes.c_int, [_CTX, ctypes.c_int32, RP_BARRIER_FN, _P]),
    "rp_schedule_static": (ctypes.c_int, [_CTX, ctypes.c_int32, ctypes.c_int64,
                                          ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]),
    "rp_schedule_static_worker": (ctypes.c_int, [_CTX, ctypes.c_int32, ctypes.c_int64, ctypes.c_int32,
                                                 ctypes.POINTER(rp_group)]),
    "rp_group_generate": (ctypes.c_int, [_CTX, ctypes.c_int32, ctypes.POINTER(rp_group)]),
    "rp_group_generate_many": (ctypes.c_int, [_CTX, ctypes.POINTER(ctypes.c_int32), ctypes.c_int32,
                                              ctypes.POINTER(rp_group)]),
    "rp_gg_release": (ctypes.c_int, [_CTX, ctypes.c_int64]),
    "rp_retire": (ctypes.c_int, [_CTX, ctypes.c_int32]),
    "rp_step": (ctypes.c_int, [_CTX, ctypes.c_int32, _P, ctypes.c_float]),
    "rp_step_bf16": (ctypes.c_int, [_CTX, ctypes.c_int32, _P, ctypes.c_float]),
    "rp_step_momentum": (ctypes.c_int, [_CTX, ctypes.c_int32, _P, ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                         _P]),
    "rp_preduce": (ctypes.c_int, [_CTX, ctypes.c_int32, ctypes.POINTER(rp_group)]),
    "rp_barrier_free_wait": (ctypes.c_int, [_CTX, ctypes.c_int32, ctypes.c_int64]),
    "rp_batch_begin": (ctypes.c_int, [_CTX]),
    "rp_batch_end": (ctypes.c_int, [_CTX]),
    "rp_timing_read": (ctypes.c_int, [_CTX, ctypes.POINTER(rp_timing)]),
    "rp_check": (ctypes.c_int, [_CTX]),
    "rp_set_compute_delay": (ctypes.c_int, [_CTX, ctypes.c_int32, ctypes.c_int64]),
    "rp_timing_records": (ctypes.c_int, [_CTX, ctypes.POINTER(rp_launch_record), ctypes.c_int32,
                                         ctypes.POINTER(ctypes.c_int32)]),
    "rp_bench_presum": (ctypes.c_int, [ctypes.POINTER(_P), ctypes.POINTER(_P), ctypes.c_int32, ctypes.c_int64,
                                       ctypes.c_float, _P, _P]),
    "rp_bench_scatter_mean": (ctypes.c_int, [_P, ctypes.c_int64, ctypes.c_float, ctypes.POINTER(_P),
                                             ctypes.c_int32, _P]),
    "rp_stats_get": (ctypes.c_int, [_CTX, ctypes.POINTER(rp_stats)]),
    "rp_trace_open": (ctypes.c_int, [_CTX, ctypes.c_char_p]),
    "rp_last_error": (ctypes.c_char_p, []),
    "rp_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "rp_abi_version": (ctypes.c_int, []),
    "rp_compute_delay": (ctypes.c_int, [_P, ctypes.c_int64]),
    "rp_fill_xi": (ctypes.c_int, [_P, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                  ctypes.c_uint64, _P]),
    "rp_lockstep_run": (ctypes.c_int, [_CTX, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_float,
                                       ctypes.c_int32]),
}
EXPORTED_SYMBOLS = tuple(_SIGNATURES)

lib = None


def load_library(path=None):
    """Load librp.so (raises OSError if it was not built: there is no fallback)."""
    global lib
    if lib is not None and path is None:
        return lib
    p = path or library_path()
    if not os.path.exists(p):
        raise OSError(f"librp.so not found at {p}: run `make -C paper_1909_08029_b200` "
                      "or __graft_entry__.build(); there is no CPU fallback")
    handle = ctypes.CDLL(p)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    if handle.rp_abi_version() != 1:
        raise OSError("librp ABI version mismatch")
    lib = handle
    return lib


def _check(status, func):
    if status != RP_OK:
        msg = load_library().rp_last_error()
        raise RPError(status, func, (msg or b"").decode(errors="replace"))
    return status


def _ptr(v):
    if v is None:
        return None
    if hasattr(v, "data_ptr"):
        return ctypes.c_void_p(v.data_ptr())
    return ctypes.c_void_p(int(v))


# ---- same-named functions ----------------------------------------------------------

def rp_init(cfg):
    L = load_library()
    out = _CTX()
    _check(L.rp_init(ctypes.byref(cfg), ctypes.byref(out)), "rp_init")
    return out


def rp_finalize(ctx):
    _check(load_library().rp_finalize(ctx), "rp_finalize")


def rp_bind_worker(ctx, w, x, g=None):
    _check(load_library().rp_bind_worker(ctx, w, _ptr(x), _ptr(g)), "rp_bind_worker")


def rp_worker_stream(ctx, w):
    out = _P()
    _check(load_library().rp_worker_stream(ctx, w, ctypes.byref(out)), "rp_worker_stream")
    return out.value or 0


def rp_set_worker_stream(ctx, w, stream):
    _check(load_library().rp_set_worker_stream(ctx, w, _ptr(stream)), "rp_set_worker_stream")


def rp_peer_export(ctx):
    """Returns this rank's rp_peer_info as bytes (to exchange between ranks)."""
    info = rp_peer_info()
    _check(load_library().rp_peer_export(ctx, ctypes.byref(info)), "rp_peer_export")
    return bytes(info)


def rp_peer_import(ctx, records):
    """records: list of rp_peer_export() byte strings, one per rank (any order)."""
    arr = (rp_peer_info * len(records))()
    for i, b in enumerate(records):
        ctypes.memmove(ctypes.byref(arr[i]), b, ctypes.sizeof(rp_peer_info))
    _check(load_library().rp_peer_import(ctx, arr, len(records)), "rp_peer_import")


def rp_nvls_supported(ctx):
    out = ctypes.c_int32()
    _check(load_library().rp_nvls_supported(ctx, ctypes.byref(out)), "rp_nvls_supported")
    return bool(out.value)


def rp_nvls_enable(ctx, min_gpus, barrier):
    """barrier(status) -> bool: collective; True iff every rank passed status == 0."""
    def _cb(_user, status):
        try:
            return 0 if barrier(int(status)) else 1
        except Exception:  # a Python exception must not cross the C boundary
            return 1
    cb = RP_BARRIER_FN(_cb)
    _check(load_library().rp_nvls_enable(ctx, min_gpus, cb, None), "rp_nvls_enable")


def rp_schedule_static(ctx, rule, step, world):
    arr = (ctypes.c_int32 * world)()
    ng = ctypes.c_int32()
    _check(load_library().rp_schedule_static(ctx, rule, step, arr, ctypes.byref(ng)), "rp_schedule_static")
    return [int(v) for v in arr], int(ng.value)


def rp_schedule_static_worker(ctx, rule, step, w):
    g = rp_group()
    _check(load_library().rp_schedule_static_worker(ctx, rule, step, w, ctypes.byref(g)),
           "rp_schedule_static_worker")
    return g


def rp_group_generate(ctx, w):
    g = rp_group()
    try:
        _check(load_library().rp_group_generate(ctx, w, ctypes.byref(g)), "rp_group_generate")
    except RPError as e:
        e.group = g            # RP_EAGAIN: the group waiting in the pending queue
        raise
    return g


def rp_group_generate_many(ctx, workers):
    n = len(workers)
    arr = (ctypes.c_int32 * n)(*workers)
    out = (rp_group * n)()
    _check(load_library().rp_group_generate_many(ctx, arr, n, out), "rp_group_generate_many")
    return list(out)


def rp_gg_release(ctx, seq):
    _check(load_library().rp_gg_release(ctx, seq), "rp_gg_release")


def rp_retire(ctx, w):
    _check(load_library().rp_retire(ctx, w), "rp_retire")


def rp_step(ctx, w, grad, lr):
    _check(load_library().rp_step(ctx, w, _ptr(grad), ctypes.c_float(lr)), "rp_step")


def rp_step_bf16(ctx, w, grad, lr):
    _check(load_library().rp_step_bf16(ctx, w, _ptr(grad), ctypes.c_float(lr)), "rp_step_bf16")


def rp_bind_worker_bf16(ctx, w, x, g=None):
    _check(load_library().rp_bind_worker_bf16(ctx, w, _ptr(x), _ptr(g)), "rp_bind_worker_bf16")


def rp_step_momentum(ctx, w, grad, lr, momentum, weight_decay, v):
    _check(load_library().rp_step_momentum(ctx, w, _ptr(grad), ctypes.c_float(lr), ctypes.c_float(momentum),
                                           ctypes.c_float(weight_decay), _ptr(v)), "rp_step_momentum")


def rp_preduce(ctx, w, group):
    _check(load_library().rp_preduce(ctx, w, ctypes.byref(group)), "rp_preduce")


def rp_barrier_free_wait(ctx, w, timeout_us):
    _check(load_library().rp_barrier_free_wait(ctx, w, timeout_us), "rp_barrier_free_wait")


def rp_batch_begin(ctx):
    _check(load_library().rp_batch_begin(ctx), "rp_batch_begin")


def rp_batch_end(ctx):
    _check(load_library().rp_batch_end(ctx), "rp_batch_end")


def rp_lockstep_run(ctx, rule, t0, steps, lr, section_length=1):
    _check(load_library().rp_lockstep_run(ctx, rule, t0, steps, lr, section_length), "rp_lockstep_run")


def rp_timing_read(ctx):
    t = rp_timing()
    _check(load_library().rp_timing_read(ctx, ctypes.byref(t)), "rp_timing_read")
    return t.as_dict()


def rp_timing_records(ctx, cap=1 << 16):
    """Per-launch records (RP_FLAG_TIMING), oldest first; drops them from the context."""
    arr = (rp_launch_record * cap)()
    n = ctypes.c_int32()
    _check(load_library().rp_timing_records(ctx, arr, cap, ctypes.byref(n)), "rp_timing_records")
    return [{"ms": r.ms, "bytes_hbm": r.bytes_hbm, "bytes_nvlink": r.bytes_nvlink, "batch": r.batch,
             "cross": bool(r.cross)} for r in arr[:n.value]]


def rp_bench_presum(xs, gs, n, lr, out, stream=0):
    """NCCL-baseline helper: out = left fold of fl(x_i - fl(lr g_i)) (not the method's path)."""
    m = len(xs)
    X = (_P * m)(*[_ptr(v).value for v in xs])
    G = (_P * m)(*[_ptr(v).value for v in gs])
    _check(load_library().rp_bench_presum(X, G, m, n, ctypes.c_float(lr), _ptr(out), _ptr(stream)),
           "rp_bench_presum")


def rp_bench_scatter_mean(s, n, k, xs, stream=0):
    """NCCL-baseline helper: x_i = fl(s / k) for every member (not the method's path)."""
    m = len(xs)
    X = (_P * m)(*[_ptr(v).value for v in xs])
    _check(load_library().rp_bench_scatter_mean(_ptr(s), n, ctypes.c_float(k), X, m, _ptr(stream)),
           "rp_bench_scatter_mean")


def rp_set_compute_delay(ctx, w, ns):
    _check(load_library().rp_set_compute_delay(ctx, w, int(ns)), "rp_set_compute_delay")


def rp_check(ctx):
    _check(load_library().rp_check(ctx), "rp_check")


def rp_stats_get(ctx):
    s = rp_stats()
    _check(load_library().rp_stats_get(ctx, ctypes.byref(s)), "rp_stats_get")
    return s.as_dict()


def rp_trace_open(ctx, path):
    _check(load_library().rp_trace_open(ctx, str(path).encode()), "rp_trace_open")


def rp_fill_xi(dst, n, seed, w, t, j0=0, stream=0):
    _check(load_library().rp_fill_xi(_ptr(dst), n, seed, w, t, j0, _ptr(stream)), "rp_fill_xi")


fill_xi = rp_fill_xi


def rp_compute_delay(stream, ns):
    _check(load_library().rp_compute_delay(_ptr(stream), int(ns)), "rp_compute_delay")


compute_delay = rp_compute_delay


class Context:
    """Owns one rp_ctx. Methods map 1:1 onto the C calls."""

    def __init__(self, world, n_params, *, n_gpus=1, workers_per_gpu=None, rank=0, device=None,
                 group_size=2, c_thres=4, nodes=0, seed_gd=3, flags=0, job_id=0, dtype="f32", watchdog_s=0):
        if dtype not in ("f32", "bf16"):
            raise ValueError("dtype must be 'f32' or 'bf16'")
        cfg = rp_config()
        cfg.dtype = RP_DTYPE_BF16 if dtype == "bf16" else RP_DTYPE_F32
        self.dtype = dtype
        cfg.world = world
        cfg.n_gpus = n_gpus
        cfg.n_params = n_params
        cfg.workers_per_gpu = workers_per_gpu if workers_per_gpu else (world // n_gpus if n_gpus else world)
        cfg.rank = rank
        cfg.device = rank if device is None else device
        cfg.group_size = group_size
        cfg.c_thres = c_thres
        cfg.nodes = nodes
        cfg.seed_gd = seed_gd
        cfg.flags = flags
        cfg.job_id = job_id
        cfg.watchdog_s = watchdog_s
        self.cfg = cfg
        self.emulate = bool(flags & RP_FLAG_EMULATE)
        self.world = world
        self.n_params = n_params
        self.wpg = cfg.workers_per_gpu
        self.rank = rank
        self.handle = rp_init(cfg)

    def local_workers(self):
        if self.emulate:               # every virtual GPU's workers live in this process
            return list(range(self.world))
        return list(range(self.rank * self.wpg, (self.rank + 1) * self.wpg))

    def close(self):
        if self.handle:
            rp_finalize(self.handle)
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def bind_worker(self, w, x, g=None):
        (rp_bind_worker_bf16 if self.dtype == "bf16" else rp_bind_worker)(self.handle, w, x, g)

    def peer_export(self):
        return rp_peer_export(self.handle)

    def peer_import(self, records):
        rp_peer_import(self.handle, records)

    def peer_setup(self, group=None):
        """Exchange peer records over torch.distributed (metadata only; the data path is the
        library's own NVLink peer loads) and map every peer's replicas and flags."""
        import torch.distributed as dist
        mine = self.peer_export()
        records = [None] * dist.get_world_size(group)
        dist.all_gather_object(records, mine, group=group)
        self.peer_import(records)

    def nvls_supported(self):
        return rp_nvls_supported(self.handle)

    def nvls_enable(self, min_gpus, group=None):
        """Collective: create the multicast objects of every GPU subset of >= min_gpus GPUs
        and route those cross-GPU groups through the in-switch (NVLS) P-Reduce. The
        barrier is an all-gather of the ranks' status over torch.distributed."""
        import torch.distributed as dist

        def barrier(status):
            out = [None] * dist.get_world_size(group)
            dist.all_gather_object(out, status, group=group)
            return all(v == 0 for v in out)
        rp_nvls_enable(self.handle, min_gpus, barrier)

    def worker_stream(self, w):
        return rp_worker_stream(self.handle, w)

    def set_worker_stream(self, w, stream):
        rp_set_worker_stream(self.handle, w, stream)

    def schedule_static(self, rule, step):
        return rp_schedule_static(self.handle, rule, step, self.world)

    def schedule_static_worker(self, rule, step, w):
        return rp_schedule_static_worker(self.handle, rule, step, w)

    def group_generate(self, w):
        return rp_group_generate(self.handle, w)

    def group_generate_wait(self, w, timeout_s=600.0, poll_s=20e-6):
        """rp_group_generate, retrying while the random GG keeps the group pending (RP_EAGAIN)."""
        import time
        t_end = time.perf_counter() + timeout_s
        while True:
            try:
                return rp_group_generate(self.handle, w)
            except RPError as e:
                if e.status != RP_EAGAIN or time.perf_counter() > t_end:
                    raise
            time.sleep(poll_s)

    def group_generate_many(self, workers):
        return rp_group_generate_many(self.handle, workers)

    def gg_release(self, seq):
        rp_gg_release(self.handle, seq)

    def retire(self, w):
        rp_retire(self.handle, w)

    def step(self, w, grad=None, lr=0.1):
        (rp_step_bf16 if self.dtype == "bf16" else rp_step)(self.handle, w, grad, lr)

    def step_momentum(self, w, grad=None, lr=0.1, momentum=0.9, weight_decay=1e-4, v=None):
        rp_step_momentum(self.handle, w, grad, lr, momentum, weight_decay, v)

    def preduce(self, w, group):
        rp_preduce(self.handle, w, group)

    def barrier_free_wait(self, w, timeout_us=RP_WAIT_DEVICE):
        rp_barrier_free_wait(self.handle, w, timeout_us)

    def batch_begin(self):
        rp_batch_begin(self.handle)

    def batch_end(self):
        rp_batch_end(self.handle)

    def lockstep_run(self, rule, t0, steps, lr=0.1, section_length=1):
        rp_lockstep_run(self.handle, rule, t0, steps, lr, section_length)

    def timing_read(self):
        return rp_timing_read(self.handle)

    def check(self):
        rp_check(self.handle)

    def set_compute_delay(self, w, ns):
        rp_set_compute_delay(self.handle, w, ns)

    def timing_records(self):
        return rp_timing_records(self.handle)

    def stats(self):
        return rp_stats_get(self.handle)

    def trace_open(self, path):
        rp_trace_open(self.handle, path)
