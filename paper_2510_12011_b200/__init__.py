"""B200-native TorchCor monodomain step (arXiv 2510.12011).

Thin ctypes binding of ``libtcb200.so`` (C ABI in ``include/tcb200.h``): the
functions below carry the ABI's names and only marshal numpy arrays; every step
of the path runs in the library's sm_100a kernels.  There is no CPU fallback:
importing this package without the built library raises ImportError, and
``tc_create`` without a CUDA device raises TcError(TC_ECUDA).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _build

__all__ = [
    "TcError", "tc_config", "tc_step_stat", "tc_config_default", "tc_create", "tc_destroy",
    "tc_last_error", "tc_set_mesh", "tc_set_mesh_elems", "tc_set_conductivity", "tc_set_ionic_param",
    "tc_get_ionic_param", "tc_add_stimulus", "tc_set_mms", "tc_assemble", "tc_step",
    "tc_num_nodes", "tc_current_step", "tc_get_v", "tc_get_activation", "tc_state_len",
    "tc_get_state", "tc_set_state", "tc_profile", "tc_profile_read", "tc_csr_upload",
    "tc_spmv", "tc_pcg", "tc_abi_version", "tc_matrix_info", "tc_nccl_unique_id", "tc_comm_init",
    "tc_mesh_pattern", "tc_rcm", "tc_partition_plan", "tc_interior_first", "tc_set_allocator", "TorchAllocator", "tc_validate", "tc_pipeline_info", "tc_set_dirichlet", "tc_set_mms_source", "tc_step_io_repeat", "Monodomain", "LIB_PATH",
    "tc_engine_info", "tc_node_order", "tc_apply", "tc_cohort_create", "tc_cohort_step", "tc_cohort_info", "tc_cohort_set_states", "tc_cohort_get_v", "tc_cohort_destroy", "tc_cohort_last_error", "Cohort",
    "TC_ENGINE_AUTO", "TC_ENGINE_GRID", "TC_ENGINE_CLUSTER",
    "TC_ION_TT2006_EPI", "TC_ION_MS", "TC_ION_MMS", "TC_ION_CRN",
]

LIB_PATH = os.environ.get("TCB200_LIB") or _build.LIB   # override: experiment variants only
TC_OK, TC_EINVAL, TC_ENOMEM, TC_ECUDA, TC_ENCCL, TC_ESOLVER, TC_ENAN, TC_ESTATE, TC_EDEGEN, TC_EREGION = range(10)
STATUS_NAMES = ["TC_OK", "TC_EINVAL", "TC_ENOMEM", "TC_ECUDA", "TC_ENCCL", "TC_ESOLVER", "TC_ENAN",
                "TC_ESTATE", "TC_EDEGEN", "TC_EREGION"]
TC_ION_TT2006_EPI, TC_ION_MS, TC_ION_MMS, TC_ION_CRN = 0, 1, 2, 3
MODELS = {"tt2006": TC_ION_TT2006_EPI, "ms": TC_ION_MS, "mms": TC_ION_MMS, "crn": TC_ION_CRN}
TC_ENGINE_AUTO, TC_ENGINE_GRID, TC_ENGINE_CLUSTER, TC_ENGINE_CLUSTER_STREAMING = 0, 1, 2, 3
ENGINES = {"auto": TC_ENGINE_AUTO, "grid": TC_ENGINE_GRID, "cluster": TC_ENGINE_CLUSTER,
           "cluster_streaming": TC_ENGINE_CLUSTER_STREAMING}


class tc_config(C.Structure):
    _fields_ = [("theta", C.c_double), ("dt", C.c_double), ("chi", C.c_double), ("cm", C.c_double),
                ("abs_tol", C.c_double), ("rel_tol", C.c_double), ("max_iters", C.c_int32),
                ("rel_mode", C.c_int32), ("model", C.c_int32), ("fail_budget", C.c_int32),
                ("lat_threshold", C.c_double), ("lrt_threshold", C.c_double),
                ("use_rcm", C.c_int32), ("pcg_variant", C.c_int32),
                ("partitions", C.c_int32), ("check_every", C.c_int32),
                ("peer", C.c_int32), ("engine", C.c_int32), ("device_setup", C.c_int32),
                ("peer_timeout_s", C.c_int32)]


class tc_step_stat(C.Structure):
    _fields_ = [("iters", C.c_int32), ("converged", C.c_int32), ("znorm", C.c_double)]


STAT_DTYPE = np.dtype([("iters", np.int32), ("converged", np.int32), ("znorm", np.float64)])


class TcError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        name = STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else str(status)
        super().__init__(f"{name}: {msg}")


def _load():
    if LIB_PATH == _build.LIB and _build.stale():
        try:  # in-tree rebuild when the sources are newer than the library
            _build.build()
        except Exception as e:  # no fallback: fail loudly
            raise ImportError(f"{LIB_PATH} is missing or stale and nvcc failed: {e}") from e
    L = C.CDLL(LIB_PATH)
    P, I32, I64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    sig = {
        "tc_config_default": ([P], None),
        "tc_create": ([P, C.c_int, P, P], I32),
        "tc_destroy": ([P], I32),
        "tc_last_error": ([P], C.c_char_p),
        "tc_set_mesh": ([P, I64, P, I64, P, P, P], I32),
        "tc_set_mesh_elems": ([P, I64, P, I64, I32, P, P, P], I32),
        "tc_set_conductivity": ([P, I32, P, P, P], I32),
        "tc_set_ionic_param": ([P, C.c_char_p, D], I32),
        "tc_get_ionic_param": ([P, C.c_char_p, P], I32),
        "tc_add_stimulus": ([P, I64, P, D, D, D], I32),
        "tc_set_mms": ([P, D, D, D, D, I64, P], I32),
        "tc_assemble": ([P], I32),
        "tc_step": ([P, I64, P], I32),
        "tc_num_nodes": ([P], I64),
        "tc_current_step": ([P], I64),
        "tc_get_v": ([P, P], I32),
        "tc_get_activation": ([P, P, P], I32),
        "tc_state_len": ([P], I64),
        "tc_get_state": ([P, P, I64], I32),
        "tc_set_state": ([P, P, I64], I32),
        "tc_step_io": ([P, I64, P, I64, P, P], I32),
        "tc_profile": ([P, C.c_int], I32),
        "tc_profile_read": ([P, P, C.c_int], I32),
        "tc_matrix_info": ([P, P], I32),
        "tc_csr_upload": ([P, I32, I64, P, P, P], I32),
        "tc_spmv": ([P, P, P], I32),
        "tc_pcg": ([P, P, P, P, P], I32),
        "tc_abi_version": ([], I32),
        "tc_nccl_unique_id": ([P], I32),
        "tc_comm_init": ([P, C.c_int, C.c_int, P], I32),
        "tc_engine_info": ([P, P], I32),
        "tc_apply": ([P, I32, P, P], I32),
        "tc_node_order": ([P, P], I32),
        "tc_cohort_create": ([P, I32, I32, I32, P], I32),
        "tc_cohort_step": ([P, I64, P], I32),
        "tc_cohort_info": ([P, P], I32),
        "tc_cohort_set_states": ([P, I64, P, P], I32),
        "tc_cohort_get_v": ([P, I64, P, P], I32),
        "tc_cohort_last_error": ([P], C.c_char_p),
        "tc_cohort_destroy": ([P], I32),
        "tc_mesh_pattern": ([I64, I64, P, P, P], I32),
        "tc_rcm": ([I64, P, P, P], I32),
        "tc_partition_plan": ([I64, P, P, I32, I32, P, P, P, P, P, P, P], I32),
        "tc_interior_first": ([I64, P, P, I32, P, P], I32),
        "tc_set_allocator": ([P, P, P, P], I32),
        "tc_validate": ([P, P], I32),
        "tc_set_dirichlet": ([P, I64, P], I32),
        "tc_set_mms_source": ([P, C.c_double, C.c_double, C.c_double, C.c_double], I32),
        "tc_pipeline_info": ([P, P], I32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    return L


_L = _load()


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.int32)


def _check(ctx, st):
    if st != TC_OK:
        raise TcError(st, tc_last_error(ctx))


# ---------------------------------------------------------------- ABI, same names
def tc_abi_version() -> int:
    return _L.tc_abi_version()


def tc_config_default(**overrides) -> tc_config:
    cfg = tc_config()
    _L.tc_config_default(C.byref(cfg))
    for k, v in overrides.items():
        if k == "model" and isinstance(v, str):
            v = MODELS[v]
        if k == "engine" and isinstance(v, str):
            v = ENGINES[v]
        setattr(cfg, k, v)
    return cfg


def tc_create(cfg: tc_config, device: int = 0, stream: int = 0):
    out = C.c_void_p()
    st = _L.tc_create(C.byref(cfg), device, C.c_void_p(stream or None), C.byref(out))
    if st != TC_OK:
        raise TcError(st, "tc_create failed (no usable CUDA device?)")
    return out


def tc_destroy(ctx) -> None:
    _L.tc_destroy(ctx)


def tc_last_error(ctx) -> str:
    m = _L.tc_last_error(ctx)
    return m.decode() if m else ""


def tc_set_mesh(ctx, xyz, tets, region=None, fibre=None) -> None:
    """Tetrahedra (n_tets, 4); a (n_elems, 3) array is routed to tc_set_mesh_elems."""
    tets = _i32(tets)
    if tets.ndim == 2 and tets.shape[1] == 3:
        return tc_set_mesh_elems(ctx, xyz, tets, region, fibre)
    xyz, region, fibre = _f64(xyz), _i32(region), _f64(fibre)
    _check(ctx, _L.tc_set_mesh(ctx, xyz.shape[0], _ptr(xyz), tets.shape[0], _ptr(tets),
                               _ptr(region), _ptr(fibre)))


def tc_set_mesh_elems(ctx, xyz, elems, region=None, fibre=None) -> None:
    """Elements with 3 (surface triangles) or 4 (tetrahedra) nodes: (n_elems, k)."""
    xyz, elems, region, fibre = _f64(xyz), _i32(elems), _i32(region), _f64(fibre)
    k = elems.shape[1] if elems.ndim == 2 else 0
    _check(ctx, _L.tc_set_mesh_elems(ctx, xyz.shape[0], _ptr(xyz), elems.shape[0], k,
                                     _ptr(elems), _ptr(region), _ptr(fibre)))


def tc_set_conductivity(ctx, ids, sigma_l, sigma_t) -> None:
    ids, sl, st = _i32(ids), _f64(sigma_l), _f64(sigma_t)
    _check(ctx, _L.tc_set_conductivity(ctx, ids.shape[0], _ptr(ids), _ptr(sl), _ptr(st)))


def tc_set_ionic_param(ctx, name: str, value: float) -> None:
    _check(ctx, _L.tc_set_ionic_param(ctx, name.encode(), float(value)))


def tc_get_ionic_param(ctx, name: str) -> float:
    v = C.c_double()
    _check(ctx, _L.tc_get_ionic_param(ctx, name.encode(), C.byref(v)))
    return v.value


def tc_add_stimulus(ctx, nodes, t_start, duration, amplitude) -> None:
    nodes = _i32(nodes)
    _check(ctx, _L.tc_add_stimulus(ctx, nodes.shape[0], _ptr(nodes), t_start, duration, amplitude))


def tc_set_mms(ctx, k, w1, w2, lam, dirichlet_nodes) -> None:
    nodes = _i32(dirichlet_nodes)
    _check(ctx, _L.tc_set_mms(ctx, k, w1, w2, lam, nodes.shape[0], _ptr(nodes)))


def tc_set_dirichlet(ctx, nodes) -> None:
    nodes = _i32(nodes)
    _check(ctx, _L.tc_set_dirichlet(ctx, nodes.shape[0], _ptr(nodes)))


def tc_set_mms_source(ctx, k, w1, w2, lam) -> None:
    _check(ctx, _L.tc_set_mms_source(ctx, k, w1, w2, lam))


def tc_assemble(ctx) -> None:
    _check(ctx, _L.tc_assemble(ctx))


def tc_step(ctx, n_steps: int, want_stats: bool = True):
    stats = np.zeros(n_steps, STAT_DTYPE) if want_stats else None
    _check(ctx, _L.tc_step(ctx, n_steps, _ptr(stats)))
    return stats


def tc_num_nodes(ctx) -> int:
    return _L.tc_num_nodes(ctx)


def tc_current_step(ctx) -> int:
    return _L.tc_current_step(ctx)


def tc_get_v(ctx, out=None):
    out = np.empty(tc_num_nodes(ctx)) if out is None else out
    _check(ctx, _L.tc_get_v(ctx, _ptr(out)))
    return out


def tc_get_activation(ctx):
    n = tc_num_nodes(ctx)
    lat, lrt = np.empty(n), np.empty(n)
    _check(ctx, _L.tc_get_activation(ctx, _ptr(lat), _ptr(lrt)))
    return lat, lrt


def tc_state_len(ctx) -> int:
    return _L.tc_state_len(ctx)


def tc_get_state(ctx, out=None):
    m = tc_state_len(ctx)
    out = np.empty(m) if out is None else out
    _check(ctx, _L.tc_get_state(ctx, _ptr(out), m))
    return out


def tc_set_state(ctx, buf) -> None:
    if not (isinstance(buf, np.ndarray) and buf.dtype == np.float64 and buf.flags.c_contiguous):
        buf = _f64(buf)
    _check(ctx, _L.tc_set_state(ctx, _ptr(buf), buf.shape[0]))


def tc_step_io(ctx, states, v_out, want_stats: bool = False):
    """states: (n_steps, >= tc_state_len) float64 host array (pinned for overlap);
    v_out: (n_steps, n_nodes) float64 host array, filled with V^{k+1} of each."""
    if not (isinstance(states, np.ndarray) and states.dtype == np.float64 and states.ndim == 2
            and states.strides[1] == 8):
        raise ValueError("states: 2-D float64 array with contiguous rows")
    if not (isinstance(v_out, np.ndarray) and v_out.dtype == np.float64 and v_out.flags.c_contiguous
            and v_out.shape == (states.shape[0], tc_num_nodes(ctx))):
        raise ValueError("v_out: C-contiguous float64 array (n_steps, n_nodes)")
    m = states.shape[0]
    stats = np.zeros(m, STAT_DTYPE) if want_stats else None
    _check(ctx, _L.tc_step_io(ctx, m, _ptr(states), states.strides[0] // 8, _ptr(v_out), _ptr(stats)))
    return stats


def tc_step_io_repeat(ctx, state, v_out, n_steps: int, want_stats: bool = False):
    """n_steps identical one-step problems from ONE host state (tc_step_io with
    stride 0): the state is copied host -> device and V^{k+1} device -> host once
    per problem; v_out (n_nodes) holds the last result."""
    if not (isinstance(state, np.ndarray) and state.dtype == np.float64 and state.flags.c_contiguous
            and state.ndim == 1 and state.shape[0] >= tc_state_len(ctx)):
        raise ValueError("state: contiguous float64 array of tc_state_len")
    if not (isinstance(v_out, np.ndarray) and v_out.dtype == np.float64 and v_out.flags.c_contiguous
            and v_out.shape == (tc_num_nodes(ctx),)):
        raise ValueError("v_out: contiguous float64 array of n_nodes")
    stats = np.zeros(n_steps, STAT_DTYPE) if want_stats else None
    _check(ctx, _L.tc_step_io(ctx, n_steps, _ptr(state), 0, _ptr(v_out), _ptr(stats)))
    return stats


def tc_profile(ctx, enable: bool = True) -> None:
    _check(ctx, _L.tc_profile(ctx, int(enable)))


def tc_profile_read(ctx, reset: bool = False):
    out = np.zeros(6)
    _check(ctx, _L.tc_profile_read(ctx, _ptr(out), int(reset)))
    return dict(ionic_ms=out[0], pcg_ms=out[1], other_ms=out[2], iters=out[3], steps=out[4],
                launches=float(out[5]))   # kernel launches (cohort members' shares of a cluster launch are fractions)


def tc_matrix_info(ctx) -> dict:
    out = np.zeros(11, np.int64)
    _check(ctx, _L.tc_matrix_info(ctx, _ptr(out)))
    return dict(n=int(out[0]), nnz=int(out[1]), nnz_pad=int(out[2]), nslices=int(out[3]),
                pcg_grid=int(out[4]), wide_slices=int(out[5]), partitions=int(out[6]),
                ghosts=int(out[7]), path=["persistent", "split", "peer"][int(out[8])],
                peer_ctas=int(out[9]), pcg_variant=int(out[10]))


def tc_nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    st = _L.tc_nccl_unique_id(buf)
    if st != TC_OK:
        raise TcError(st, "ncclGetUniqueId failed (NCCL not loadable?)")
    return bytes(buf)


def tc_comm_init(ctx, rank: int, world: int, unique_id: bytes) -> None:
    buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
    _check(ctx, _L.tc_comm_init(ctx, rank, world, buf))


def tc_apply(ctx, which: int, x):
    """A x (which 0) or K x (which 1), original node order."""
    x = _f64(x)
    y = np.empty_like(x)
    _check(ctx, _L.tc_apply(ctx, which, _ptr(x), _ptr(y)))
    return y


def tc_node_order(ctx):
    perm = np.empty(tc_num_nodes(ctx), np.int32)
    _check(ctx, _L.tc_node_order(ctx, _ptr(perm)))
    return perm


def tc_engine_info(ctx) -> dict:
    out = np.zeros(4, np.int64)
    _check(ctx, _L.tc_engine_info(ctx, _ptr(out)))
    return dict(engine={1: "grid", 2: "cluster"}[int(out[0])], cluster_size=int(out[1]),
                smem_per_cta=int(out[2]), resident_clusters=int(out[3]))


# ---------------------------------------------------------------- cohorts
def tc_cohort_create(members, cluster_size: int = 0, resident: int = 1):
    """members: contexts (assembled, single partition, same device and model)."""
    arr = (C.c_void_p * len(members))(*[m.value if isinstance(m, C.c_void_p) else m for m in members])
    out = C.c_void_p()
    st = _L.tc_cohort_create(arr, len(members), cluster_size, int(resident), C.byref(out))
    if st != TC_OK:
        raise TcError(st, tc_last_error(members[0]) if members else "tc_cohort_create")
    return out


def tc_cohort_step(co, n_steps: int, count: int | None = None, want_stats: bool = True):
    """-> stats (count, n_steps) structured array, member-major (or None)."""
    stats = None
    if want_stats:
        if count is None:
            count = tc_cohort_info(co)["members"]
        stats = np.zeros((count, n_steps), STAT_DTYPE)
    st = _L.tc_cohort_step(co, n_steps, _ptr(stats))
    if st != TC_OK:
        m = _L.tc_cohort_last_error(co)
        raise TcError(st, m.decode() if m else "")
    return stats


def _ptr_array(arrs):
    for a in arrs:
        if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous):
            raise ValueError("cohort I/O: contiguous float64 arrays")
    ptrs = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    lens = np.array([a.size for a in arrs], np.int64)
    return len(arrs), ptrs, lens


def _co_check(co, st):
    if st != TC_OK:
        m = _L.tc_cohort_last_error(co)
        raise TcError(st, m.decode() if m else "")


def tc_cohort_set_states(co, bufs) -> None:
    """bufs: one tc_set_state-layout float64 host array per member (member order);
    the library checks the count and every length."""
    cnt, ptrs, lens = _ptr_array(bufs)
    _co_check(co, _L.tc_cohort_set_states(co, cnt, ptrs, _ptr(lens)))


def tc_cohort_get_v(co, outs) -> None:
    """outs: one float64 host array of n_nodes per member, filled with V^k."""
    cnt, ptrs, lens = _ptr_array(outs)
    _co_check(co, _L.tc_cohort_get_v(co, cnt, ptrs, _ptr(lens)))


def tc_cohort_info(co) -> dict:
    out = np.zeros(6, np.int32)
    st = _L.tc_cohort_info(co, _ptr(out))
    if st != TC_OK:
        raise TcError(st, "tc_cohort_info")
    return dict(members=int(out[0]), cluster_size=int(out[1]), resident_clusters=int(out[2]),
                smem_per_cta=int(out[3]), compact=bool(out[4]), dense=bool(out[5]))


def tc_cohort_last_error(co) -> str:
    m = _L.tc_cohort_last_error(co)
    return m.decode() if m else ""


def tc_cohort_destroy(co) -> None:
    _L.tc_cohort_destroy(co)


# ---------------------------------------------------------------- host-only helpers
def tc_mesh_pattern(n: int, tets):
    tets = _i32(tets)
    rowptr = np.zeros(n + 1, np.int64)
    st = _L.tc_mesh_pattern(n, tets.shape[0], _ptr(tets), _ptr(rowptr), None)
    if st != TC_OK:
        raise TcError(st, "tc_mesh_pattern")
    col = np.zeros(int(rowptr[n]), np.int32)
    _L.tc_mesh_pattern(n, tets.shape[0], _ptr(tets), _ptr(rowptr), _ptr(col))
    return rowptr, col


def tc_rcm(rowptr, col):
    rowptr = np.ascontiguousarray(rowptr, np.int64)
    col = _i32(col)
    n = rowptr.shape[0] - 1
    perm = np.zeros(n, np.int32)
    st = _L.tc_rcm(n, _ptr(rowptr), _ptr(col), _ptr(perm))
    if st != TC_OK:
        raise TcError(st, "tc_rcm")
    return perm


def tc_interior_first(rowptr, col, nparts: int):
    """-> (order[new] = old, n_interior per block) of the interior-first block order."""
    rowptr = np.ascontiguousarray(rowptr, np.int64)
    col = _i32(col)
    n = rowptr.shape[0] - 1
    order = np.zeros(n, np.int32)
    nint = np.zeros(nparts, np.int64)
    st = _L.tc_interior_first(n, _ptr(rowptr), _ptr(col), nparts, _ptr(order), _ptr(nint))
    if st != TC_OK:
        raise TcError(st, "tc_interior_first")
    return order, nint


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)


class TorchAllocator:
    """tc_set_allocator callbacks backed by torch's CUDA caching allocator
    (SURVEY 8(b)); keeps the ctypes trampolines alive and counts live blocks."""

    def __init__(self, device: int = 0):
        import torch
        self.torch, self.device, self.live = torch, device, {}

        def _alloc(nbytes, stream, user):
            try:
                p = self.torch.cuda.caching_allocator_alloc(int(nbytes), self.device, int(stream or 0))
            except Exception:
                return None
            self.live[p] = int(nbytes)
            return p

        def _free(ptr, stream, user):
            if ptr:
                self.live.pop(int(ptr), None)
                self.torch.cuda.caching_allocator_delete(int(ptr))

        self.alloc_fn = ALLOC_FN(_alloc)
        self.free_fn = FREE_FN(_free)


def tc_pipeline_info(ctx) -> dict:
    out = np.zeros(2, np.int64)
    _check(ctx, _L.tc_pipeline_info(ctx, _ptr(out)))
    return dict(chunks=int(out[0]), rows_per_chunk=int(out[1]))


def tc_validate(ctx) -> int:
    """Index audit of an assembled context (include/tcb200.h); returns the number of checked indices."""
    out = np.zeros(1, np.int64)
    _check(ctx, _L.tc_validate(ctx, _ptr(out)))
    return int(out[0])


def tc_set_allocator(ctx, allocator) -> None:
    """allocator: an object with alloc_fn / free_fn ctypes callbacks (TorchAllocator), or None."""
    if allocator is None:
        _check(ctx, _L.tc_set_allocator(ctx, None, None, None))
    else:
        _check(ctx, _L.tc_set_allocator(ctx, C.cast(allocator.alloc_fn, C.c_void_p),
                                        C.cast(allocator.free_fn, C.c_void_p), None))


def tc_partition_plan(rowptr, col, nparts: int, part: int) -> dict:
    rowptr = np.ascontiguousarray(rowptr, np.int64)
    col = _i32(col)
    n = rowptr.shape[0] - 1
    sizes = np.zeros(4, np.int64)
    st = _L.tc_partition_plan(n, _ptr(rowptr), _ptr(col), nparts, part, _ptr(sizes),
                              None, None, None, None, None, None)
    if st != TC_OK:
        raise TcError(st, "tc_partition_plan")
    ng, nn, ns, _ = (int(v) for v in sizes)
    bounds = np.zeros(nparts + 1, np.int64)
    ghosts = np.zeros(ng, np.int32)
    nbr = np.zeros(nn, np.int32)
    recv_off = np.zeros(nn + 1, np.int64)
    send_off = np.zeros(nn + 1, np.int64)
    send_g = np.zeros(ns, np.int32)
    _L.tc_partition_plan(n, _ptr(rowptr), _ptr(col), nparts, part, _ptr(sizes), _ptr(bounds),
                         _ptr(ghosts), _ptr(nbr), _ptr(recv_off), _ptr(send_off), _ptr(send_g))
    return dict(bounds=bounds, ghosts=ghosts, nbr=nbr, recv_off=recv_off, send_off=send_off,
                send_g=send_g)


def tc_csr_upload(ctx, rowptr, col, val) -> None:
    rowptr, col, val = _i32(rowptr), _i32(col), _f64(val)
    _check(ctx, _L.tc_csr_upload(ctx, rowptr.shape[0] - 1, col.shape[0], _ptr(rowptr), _ptr(col),
                                 _ptr(val)))


def tc_spmv(ctx, x):
    x = _f64(x)
    y = np.empty_like(x)
    _check(ctx, _L.tc_spmv(ctx, _ptr(x), _ptr(y)))
    return y


def tc_pcg(ctx, b, x0):
    b, x0 = _f64(b), _f64(x0)
    x = np.empty_like(b)
    rep = tc_step_stat()
    _check(ctx, _L.tc_pcg(ctx, _ptr(b), _ptr(x0), _ptr(x), C.byref(rep)))
    return x, dict(iters=rep.iters, converged=bool(rep.converged), znorm=rep.znorm)


# ---------------------------------------------------------------- convenience wrapper
class Monodomain:
    """Owning wrapper: ``Monodomain(xyz, tets, region, fibre, {tag: (sl, st)}, cfg, stimuli)``.

    ``stimuli`` are (nodes, t_start, duration, amplitude) tuples or objects with
    those attributes.  Host-side orchestration only."""

    def __init__(self, xyz, tets, region, fibre, conductivities: dict, cfg: tc_config,
                 stimuli=(), device: int = 0, stream: int = 0, mms=None, params: dict | None = None,
                 comm=None, allocator=None):
        self.ctx = tc_create(cfg, device, stream)
        self.allocator = allocator        # kept alive until close()
        try:
            if allocator is not None:
                tc_set_allocator(self.ctx, allocator)
            if comm is not None:          # (rank, world, nccl_unique_id)
                tc_comm_init(self.ctx, *comm)
            tc_set_mesh(self.ctx, xyz, tets, region, fibre)
            ids = sorted(conductivities)
            tc_set_conductivity(self.ctx, ids, [conductivities[i][0] for i in ids],
                                [conductivities[i][1] for i in ids])
            for name, v in (params or {}).items():
                tc_set_ionic_param(self.ctx, name, v)
            for s in stimuli:
                if isinstance(s, tuple):
                    nodes, t0, dur, amp = s
                else:
                    nodes, t0, dur, amp = s.nodes, s.start, s.duration, s.amplitude
                tc_add_stimulus(self.ctx, nodes, t0, dur, amp)
            if mms is not None:
                tc_set_mms(self.ctx, *mms)
            tc_assemble(self.ctx)
        except Exception:
            tc_destroy(self.ctx)
            self.ctx = None
            raise

    def step(self, n: int = 1):
        return tc_step(self.ctx, n)

    @property
    def V(self):
        return tc_get_v(self.ctx)

    def activation(self):
        return tc_get_activation(self.ctx)

    def get_state(self):
        return tc_get_state(self.ctx)

    def set_state(self, buf):
        tc_set_state(self.ctx, buf)

    def close(self):
        if self.ctx is not None:
            tc_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Cohort:
    """Owning wrapper over tc_cohort_*: ``Cohort([Monodomain, ...])``; the members
    stay usable (``m.V``, ``m.activation()``) and must outlive the cohort."""

    def __init__(self, members, cluster_size: int = 0, resident: int = 1):
        self.members = list(members)
        self.co = tc_cohort_create([m.ctx for m in self.members], cluster_size, resident)

    def step(self, n: int = 1, want_stats: bool = True):
        return tc_cohort_step(self.co, n, len(self.members), want_stats)

    def set_states(self, bufs) -> None:
        tc_cohort_set_states(self.co, bufs)

    def get_v(self, outs) -> None:
        tc_cohort_get_v(self.co, outs)

    def info(self) -> dict:
        return tc_cohort_info(self.co)

    def close(self):
        if self.co is not None:
            tc_cohort_destroy(self.co)
            self.co = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
