"""Python binding of libptdr.so -- argument marshalling only.

Every step of the decomposition runs in the CUDA kernels behind the C ABI
(include/ptdr.h).  PyTorch is used only for device memory and streams.  There
is no CPU fallback: if the shared library is missing or CUDA is unavailable the
calls raise.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, os.environ.get("PTDR_LIB_NAME", "libptdr.so"))

STRUCTURES = {
    "general": 0,
    "hermitian": 1,
    "real_symmetric": 2,
    "diagonal": 3,
    "tridiagonal": 4,
    "anti_diagonal": 5,
    "hermitian_tridiagonal": 6,
}
PTDR_OK, PTDR_EINVAL, PTDR_EUNSUPPORTED, PTDR_ENOMEM, PTDR_ECUDA = 0, 1, 2, 3, 4


class PtdrError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{msg} (status {status})")
        self.status = status


_lib = None


def lib():
    """Load libptdr.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} not found: build it with `python paper_2403_11644_b200/build.py` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        i32, u64, sz, vp = ctypes.c_int, ctypes.c_uint64, ctypes.c_size_t, ctypes.c_void_p
        L.ptdr_max_n.argtypes = [i32]
        L.ptdr_input_count.argtypes = [i32, i32]
        L.ptdr_input_count.restype = sz
        L.ptdr_output_count.argtypes = [i32, i32]
        L.ptdr_output_count.restype = sz
        L.ptdr_workspace_bytes.argtypes = [i32, i32, i32]
        L.ptdr_workspace_bytes.restype = sz
        L.ptdr_decompose.argtypes = [vp, i32, i32, vp]
        L.ptdr_decompose_async.argtypes = [vp, i32, i32, vp, vp, sz, vp]
        L.ptdr_inplace_workspace_bytes.argtypes = [i32, i32]
        L.ptdr_inplace_workspace_bytes.restype = sz
        L.ptdr_decompose_inplace_async.argtypes = [vp, i32, i32, vp, sz, vp]
        L.ptdr_decompose_inplace_async.restype = i32
        L.ptdr_decompose_matrix_layout_async.argtypes = [vp, i32, i32, vp, vp, sz, vp]
        L.ptdr_decompose_matrix_layout_async.restype = i32
        L.ptdr_decompose_host.argtypes = [vp, i32, i32, vp]
        L.ptdr_decompose_xshard_async.argtypes = [vp, i32, i32, i32, vp, vp, sz, vp]
        L.ptdr_decompose_xshard_ex_async.argtypes = [vp, i32, i32, i32, vp, vp, sz, i32, vp]
        L.ptdr_decompose_xshard_ex_async.restype = i32
        L.ptdr_decompose_zshard_async.argtypes = [vp, i32, i32, i32, i32, vp, vp, sz, vp]
        L.ptdr_decompose_zshard_async.restype = i32
        L.ptdr_band_xmask_count.argtypes = [i32, i32]
        L.ptdr_band_xmask_count.restype = sz
        L.ptdr_band_xmasks.argtypes = [i32, i32, ctypes.POINTER(ctypes.c_uint64), sz]
        L.ptdr_band_xmasks.restype = i32
        L.ptdr_band_workspace_bytes.argtypes = [i32, i32]
        L.ptdr_band_workspace_bytes.restype = sz
        L.ptdr_decompose_band_async.argtypes = [vp, i32, i32, vp, vp, sz, vp]
        L.ptdr_decompose_band_async.restype = i32
        dbl = ctypes.c_double
        L.ptdr_reconstruct_workspace_bytes.argtypes = [i32]
        L.ptdr_reconstruct_workspace_bytes.restype = sz
        L.ptdr_reconstruct_async.argtypes = [vp, i32, vp, vp, sz, vp]
        L.ptdr_reconstruct_matrix_layout_workspace_bytes.argtypes = [i32]
        L.ptdr_reconstruct_matrix_layout_workspace_bytes.restype = sz
        L.ptdr_reconstruct_matrix_layout_async.argtypes = [vp, i32, vp, vp, sz, vp]
        L.ptdr_axpby_async.argtypes = [vp, dbl, dbl, vp, dbl, dbl, vp, sz, vp]
        L.ptdr_block_diag_async.argtypes = [vp, i32, i32, vp, vp]
        L.ptdr_hermitian_augment_async.argtypes = [vp, i32, vp, vp]
        for name in ("ptdr_reconstruct_async", "ptdr_reconstruct_matrix_layout_async", "ptdr_axpby_async",
                     "ptdr_block_diag_async", "ptdr_hermitian_augment_async"):
            getattr(L, name).restype = i32
        L.ptdr_padded_workspace_bytes.argtypes = [u64, i32]
        L.ptdr_padded_workspace_bytes.restype = sz
        L.ptdr_decompose_padded_async.argtypes = [vp, u64, u64, i32, vp, vp, sz, vp]
        L.ptdr_decompose_padded_async.restype = i32
        L.ptdr_decompose_peer_async.argtypes = [ctypes.POINTER(vp), i32, i32, i32, vp, vp, sz, vp]
        L.ptdr_decompose_peer_async.restype = i32
        L.ptdr_ipc_handle_size.restype = sz
        L.ptdr_ipc_get_handle.argtypes = [vp, vp, ctypes.POINTER(u64)]
        L.ptdr_ipc_open.argtypes = [vp, ctypes.POINTER(vp)]
        L.ptdr_ipc_close.argtypes = [vp]
        for name in ("ptdr_ipc_get_handle", "ptdr_ipc_open", "ptdr_ipc_close"):
            getattr(L, name).restype = i32
        L.ptdr_generated_workspace_bytes.argtypes = [i32, i32]
        L.ptdr_generated_workspace_bytes.restype = sz
        L.ptdr_decompose_generated_async.argtypes = [i32, u64, i32, i32, vp, vp, sz, vp]
        L.ptdr_decompose_generated_async.restype = i32
        L.ptdr_coefficients_async.argtypes = [vp, i32, vp, u64, vp, vp]
        L.ptdr_coefficients_async.restype = i32
        L.ptdr_coefficients_xshard_async.argtypes = [vp, i32, i32, i32, vp, u64, vp, vp]
        L.ptdr_coefficients_xshard_async.restype = i32
        L.ptdr_decompose_batched_async.argtypes = [vp, i32, i32, u64, vp, vp]
        L.ptdr_decompose_batched_async.restype = i32
        L.ptdr_generate_dense_async.argtypes = [i32, u64, i32, u64, u64, vp, vp, vp]
        L.ptdr_generate_band_async.argtypes = [i32, u64, i32, vp, vp, vp]
        L.ptdr_generate_sendblocks_async.argtypes = [i32, u64, i32, i32, i32, vp, vp, vp]
        L.ptdr_fro2_partial_count.restype = sz
        L.ptdr_sumsq_async.argtypes = [vp, u64, vp, vp]
        L.ptdr_sumsq_async.restype = i32
        L.ptdr_status_string.argtypes = [i32]
        L.ptdr_status_string.restype = ctypes.c_char_p
        L.ptdr_last_error.restype = ctypes.c_char_p
        L.ptdr_last_launch_count.restype = i32
        L.ptdr_version.restype = i32
        L.ptdr_plan_create.argtypes = [i32, i32, i32, ctypes.POINTER(vp)]
        L.ptdr_plan_decompose_host_async.argtypes = [vp, vp, vp]
        L.ptdr_plan_wait.argtypes = [vp]
        L.ptdr_plan_launch_count.argtypes = [vp]
        L.ptdr_plan_launch_count.restype = i32
        L.ptdr_plan_destroy.argtypes = [vp]
        for name in ("ptdr_plan_create", "ptdr_plan_decompose_host_async", "ptdr_plan_wait",
                     "ptdr_plan_destroy"):
            getattr(L, name).restype = i32
        for name in ("ptdr_decompose", "ptdr_decompose_async", "ptdr_decompose_host",
                     "ptdr_decompose_xshard_async", "ptdr_generate_dense_async",
                     "ptdr_generate_band_async", "ptdr_generate_sendblocks_async"):
            getattr(L, name).restype = i32
        _lib = L
    return _lib


def _check(status: int, what: str):
    if status != PTDR_OK:
        L = lib()
        raise PtdrError(status, f"{what}: {L.ptdr_status_string(status).decode()}: "
                                f"{L.ptdr_last_error().decode()}")


def _structure(s) -> int:
    return STRUCTURES[s] if isinstance(s, str) else int(s)


def _stream_ptr(stream):
    import torch

    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def input_count(n: int, structure="general") -> int:
    return int(lib().ptdr_input_count(n, _structure(structure)))


def output_count(n: int, structure="general") -> int:
    return int(lib().ptdr_output_count(n, _structure(structure)))


def workspace_bytes(n: int, structure="general", world: int = 1) -> int:
    v = int(lib().ptdr_workspace_bytes(n, _structure(structure), world))
    if v == ctypes.c_size_t(-1).value:
        raise PtdrError(PTDR_EINVAL, f"invalid (n={n}, structure={structure}, world={world})")
    return v


def last_launch_count() -> int:
    return int(lib().ptdr_last_launch_count())


def _require_cuda_c128(t, name, count=None, device=None):
    """Type, size and device checks before any ABI call: the C ABI takes raw pointers and
    cannot check buffer sizes itself."""
    import torch

    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != torch.complex128 or not t.is_contiguous():
        raise TypeError(f"{name} must be contiguous complex128")
    if count is not None and t.numel() != count:
        raise ValueError(f"{name} holds {t.numel()} elements, expected {count}")
    if device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device}")


def _require_workspace(ws, nbytes, device):
    import torch

    if not isinstance(ws, torch.Tensor) or not ws.is_cuda or not ws.is_contiguous():
        raise TypeError("workspace must be a contiguous CUDA tensor")
    if ws.device != device:
        raise ValueError(f"workspace is on {ws.device}, expected {device}")
    if ws.numel() * ws.element_size() < nbytes:
        raise ValueError(f"workspace holds {ws.numel() * ws.element_size()} bytes, needs {nbytes}")


def _keep_for_stream(stream, *tensors):
    """Temporaries allocated here come from torch's caching allocator, which orders their
    reuse on the CURRENT stream only.  When the kernels run on another stream, record that
    stream on them so the blocks are not handed out again before the kernels finish."""
    import torch

    if stream is None:
        return
    if stream.cuda_stream == torch.cuda.current_stream(stream.device).cuda_stream:
        return
    for t in tensors:
        if t is not None:
            t.record_stream(stream)


def _pow2_exponent(N: int, what: str) -> int:
    n = int(N).bit_length() - 1
    if N < 1 or (1 << n) != N:
        raise ValueError(f"{what} must be a power of two (got {N}); use decompose_padded for other sizes")
    return n


def n_of(A, structure="general") -> int:
    """n of an input array: dense [2^n, 2^n]; DIAGONAL / ANTI_DIAGONAL [2^n];
    TRIDIAGONAL [3, 2^n] (or 3 * 2^n elements); HERMITIAN_TRIDIAGONAL [2, 2^n] (main, sup).
    Torch tensors or numpy arrays."""
    s = _structure(structure)
    ndim = len(A.shape)
    numel = 1
    for d in A.shape:
        numel *= int(d)
    if s <= 2:
        N = A.shape[-1]
        if ndim != 2 or A.shape[0] != N:
            raise ValueError("dense A must be 2^n x 2^n")
        return _pow2_exponent(N, "the matrix size")
    if s in (3, 5):
        if ndim != 1:
            raise ValueError("DIAGONAL / ANTI_DIAGONAL input is a 1-D array of 2^n elements")
        return _pow2_exponent(numel, "the band length")
    if s == 4:
        if numel % 3 != 0 or (ndim == 2 and A.shape[0] != 3) or ndim > 2:
            raise ValueError("TRIDIAGONAL input is [3, 2^n] (sub, main, sup)")
        return _pow2_exponent(numel // 3, "the band length")
    if s == 6:
        if numel % 2 != 0 or (ndim == 2 and A.shape[0] != 2) or ndim > 2:
            raise ValueError("HERMITIAN_TRIDIAGONAL input is [2, 2^n] (main, sup)")
        return _pow2_exponent(numel // 2, "the band length")
    raise ValueError(f"unknown structure {structure!r}")


def alloc_workspace(n: int, structure="general", world: int = 1, device=None):
    import torch

    nb = workspace_bytes(n, structure, world)
    # torch's caching allocator returns >= 512-byte aligned blocks
    return torch.empty(max(nb, 1), dtype=torch.uint8, device=device if device is not None else "cuda")


def _workspace(workspace, n, structure, world, device, stream):
    """The caller's workspace (checked), or a temporary kept alive for `stream`."""
    nb = workspace_bytes(n, structure, world)
    if workspace is None:
        workspace = alloc_workspace(n, structure, world, device)
        _keep_for_stream(stream, workspace)
    else:
        _require_workspace(workspace, nb, device)
    return workspace


def _out(out, count, device, stream):
    import torch

    if out is None:
        out = torch.empty(count, dtype=torch.complex128, device=device)
        _keep_for_stream(stream, out)
    else:
        _require_cuda_c128(out, "out", count, device)
    return out


def decompose_matrix_layout(A, structure="general", out=None, workspace=None, stream=None):
    """All coefficients in the matrix layout out[z][z ^ x] = alpha(x, z) (out of place;
    ptdr_decompose_matrix_layout_async).  Returns out [2^n, 2^n]."""
    import torch

    _require_cuda_c128(A, "A")
    s = _structure(structure)
    n = n_of(A, s)
    if s > 2:
        raise ValueError("the matrix layout is for the dense structures")
    if out is None:
        out = torch.empty((1 << n, 1 << n), dtype=torch.complex128, device=A.device)
        _keep_for_stream(stream, out)
    _require_cuda_c128(out, "out", 4 ** n, A.device)
    nb = int(lib().ptdr_inplace_workspace_bytes(n, s))
    if workspace is None:
        workspace = torch.empty(max(nb, 1), dtype=torch.uint8, device=A.device)
        _keep_for_stream(stream, workspace)
    else:
        _require_workspace(workspace, nb, A.device)
    _check(lib().ptdr_decompose_matrix_layout_async(ctypes.c_void_p(A.data_ptr()), n, s,
                                                    ctypes.c_void_p(out.data_ptr()),
                                                    ctypes.c_void_p(workspace.data_ptr()),
                                                    workspace.numel() * workspace.element_size(),
                                                    _stream_ptr(stream)), "ptdr_decompose_matrix_layout_async")
    return out


def decompose(A, structure="general", out=None, workspace=None, stream=None, inplace=False):
    """All Pauli coefficients of A (CUDA complex128) via ptdr_decompose_async.

    Dense structures: A is [2^n, 2^n]; DIAGONAL: d[2^n]; TRIDIAGONAL: [3, 2^n]
    (sub, main, sup).  Returns `out` (q order, see include/ptdr.h).

    inplace=True (dense structures): A is overwritten with its coefficients in the matrix
    layout A[z][z ^ x] = alpha(x, z) (ptdr_decompose_inplace_async; matrix_index maps a
    string to its element) and A is returned -- no second 4^n buffer (n = 16 on one GPU
    in 64 GiB + 2 GiB)."""
    import torch

    _require_cuda_c128(A, "A")
    s = _structure(structure)
    n = n_of(A, s)
    if inplace:
        if out is not None:
            raise ValueError("inplace=True writes into A; do not pass out")
        nb = int(lib().ptdr_inplace_workspace_bytes(n, s))
        if nb == ctypes.c_size_t(-1).value:
            raise PtdrError(PTDR_EINVAL, f"in-place decomposition needs a dense structure (got {structure!r})")
        if workspace is None:
            workspace = torch.empty(max(nb, 1), dtype=torch.uint8, device=A.device)
            _keep_for_stream(stream, workspace)
        else:
            _require_workspace(workspace, nb, A.device)
        _check(lib().ptdr_decompose_inplace_async(ctypes.c_void_p(A.data_ptr()), n, s,
                                                  ctypes.c_void_p(workspace.data_ptr()),
                                                  workspace.numel() * workspace.element_size(),
                                                  _stream_ptr(stream)), "ptdr_decompose_inplace_async")
        return A
    _require_cuda_c128(A, "A", input_count(n, s))
    out = _out(out, output_count(n, s), A.device, stream)
    workspace = _workspace(workspace, n, s, 1, A.device, stream)
    st = lib().ptdr_decompose_async(ctypes.c_void_p(A.data_ptr()), n, s,
                                    ctypes.c_void_p(out.data_ptr()),
                                    ctypes.c_void_p(workspace.data_ptr()),
                                    workspace.numel(), _stream_ptr(stream))
    _check(st, "ptdr_decompose_async")
    return out


def decompose_host(A_host, structure="general", out_host=None):
    """End-to-end from host memory (numpy or CPU torch tensor, complex128)."""
    import numpy as np

    s = _structure(structure)
    a = A_host
    if not isinstance(a, np.ndarray):
        a = a.numpy()
    if a.dtype != np.complex128 or not a.flags.c_contiguous:
        raise TypeError("A_host must be C-contiguous complex128")
    n = n_of(a, s)
    if a.size != input_count(n, s):
        raise ValueError(f"A_host holds {a.size} elements, expected {input_count(n, s)}")
    if out_host is None:
        out_host = np.empty(output_count(n, s), dtype=np.complex128)
    o = out_host if isinstance(out_host, np.ndarray) else out_host.numpy()
    if o.dtype != np.complex128 or not o.flags.c_contiguous or o.size != output_count(n, s):
        raise ValueError(f"out_host must be C-contiguous complex128 with {output_count(n, s)} elements")
    st = lib().ptdr_decompose_host(ctypes.c_void_p(a.ctypes.data), n, s,
                                   ctypes.c_void_p(o.ctypes.data))
    _check(st, "ptdr_decompose_host")
    return out_host


class HostPlan:
    """Streaming decomposition of host-resident matrices (ptdr_plan_*, include/ptdr.h).

    ``depth`` device buffer slots; with depth >= 2 the upload of one matrix overlaps the
    download of the previous result.  Host arrays must stay untouched until ``wait()``."""

    def __init__(self, n: int, structure="general", depth: int = 2):
        self.n, self.structure, self.depth = n, _structure(structure), depth
        h = ctypes.c_void_p()
        _check(lib().ptdr_plan_create(n, self.structure, depth, ctypes.byref(h)), "ptdr_plan_create")
        self._h = h

    @staticmethod
    def _np(x):
        import numpy as np

        a = x if isinstance(x, np.ndarray) else x.numpy()
        if a.dtype != np.complex128 or not a.flags.c_contiguous:
            raise TypeError("host buffers must be C-contiguous complex128")
        return a

    def decompose_async(self, A_host, out_host):
        a, o = self._np(A_host), self._np(out_host)
        if a.size != input_count(self.n, self.structure) or o.size != output_count(self.n, self.structure):
            raise ValueError("host buffer sizes do not match the plan")
        _check(lib().ptdr_plan_decompose_host_async(self._h, ctypes.c_void_p(a.ctypes.data),
                                                    ctypes.c_void_p(o.ctypes.data)),
               "ptdr_plan_decompose_host_async")

    def wait(self):
        _check(lib().ptdr_plan_wait(self._h), "ptdr_plan_wait")

    def launch_count(self) -> int:
        return lib().ptdr_plan_launch_count(self._h)

    def close(self):
        if self._h is not None and self._h.value:
            _check(lib().ptdr_plan_destroy(self._h), "ptdr_plan_destroy")
        self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def decompose_xshard(A_local, n: int, rank: int, world: int, out=None, workspace=None,
                     stream=None, max_ctas: int = 0):
    """Per-rank decomposition of the X-mask shard (after the all-to-all).  max_ctas > 0
    caps the pipeline's persistent grid (SMs left to a concurrent collective)."""
    import torch

    if world < 1 or world & (world - 1) or not 0 <= rank < world:
        raise ValueError(f"invalid rank {rank} / world {world}")
    count = (1 << (2 * n)) // world
    _require_cuda_c128(A_local, "A_local", count)
    out = _out(out, count, A_local.device, stream)
    workspace = _workspace(workspace, n, "general", world, A_local.device, stream)
    st = lib().ptdr_decompose_xshard_ex_async(ctypes.c_void_p(A_local.data_ptr()), n, rank, world,
                                              ctypes.c_void_p(out.data_ptr()),
                                              ctypes.c_void_p(workspace.data_ptr()),
                                              workspace.numel(), int(max_ctas), _stream_ptr(stream))
    _check(st, "ptdr_decompose_xshard_ex_async")
    return out


def coefficients(A, qs, out=None, stream=None):
    """Coefficients of the strings qs (q order) of a dense matrix by Algorithm 2 directly
    (ptdr_coefficients_async); qs: CUDA int64/uint64 tensor or anything torch.as_tensor takes."""
    import torch

    _require_cuda_c128(A, "A")
    n = n_of(A, 0)
    q = torch.as_tensor(qs, dtype=torch.int64, device=A.device).contiguous()
    _keep_for_stream(stream, q)
    out = _out(out, q.numel(), A.device, stream)
    _check(lib().ptdr_coefficients_async(ctypes.c_void_p(A.data_ptr()), n, ctypes.c_void_p(q.data_ptr()), q.numel(),
                                         ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream)),
           "ptdr_coefficients_async")
    return out


def coefficients_xshard(A_local, n: int, rank: int, world: int, qs, out=None, stream=None):
    """Selected coefficients (global q's of rank's X-mask shard) by Algorithm 2 on the shard
    A_local [2^n, 2^n / world] (ptdr_coefficients_xshard_async); strings outside the shard
    give NaN."""
    import torch

    _require_cuda_c128(A_local, "A_local", (1 << (2 * n)) // world)
    q = torch.as_tensor(qs, dtype=torch.int64, device=A_local.device).contiguous()
    _keep_for_stream(stream, q)
    out = _out(out, q.numel(), A_local.device, stream)
    _check(lib().ptdr_coefficients_xshard_async(ctypes.c_void_p(A_local.data_ptr()), n, rank, world,
                                                ctypes.c_void_p(q.data_ptr()), q.numel(),
                                                ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream)),
           "ptdr_coefficients_xshard_async")
    return out


def decompose_batched(A, structure="general", out=None, stream=None):
    """A batch of small dense matrices [batch, 2^n, 2^n] (n <= 10) in one launch
    (ptdr_decompose_batched_async) -> [batch, 4^n] coefficients."""
    import torch

    _require_cuda_c128(A, "A")
    if A.dim() != 3 or A.shape[1] != A.shape[2]:
        raise ValueError("A must be [batch, 2^n, 2^n]")
    B, N = A.shape[0], A.shape[1]
    n = N.bit_length() - 1
    if (1 << n) != N:
        raise ValueError("2^n x 2^n matrices")
    s = _structure(structure)
    if out is None:
        out = torch.empty((B, 4 ** n), dtype=torch.complex128, device=A.device)
        _keep_for_stream(stream, out)
    _require_cuda_c128(out, "out", B * 4 ** n, A.device)
    _check(lib().ptdr_decompose_batched_async(ctypes.c_void_p(A.data_ptr()), n, s, B,
                                              ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream)),
           "ptdr_decompose_batched_async")
    return out


def decompose_padded(A, structure="general", out=None, workspace=None, stream=None):
    """Any m x m dense matrix (a CUDA complex128 view with unit column stride, any row
    pitch) decomposed as the top-left block of the zero-padded 2^n x 2^n matrix,
    n = max(1, ceil(log2 m)) (ptdr_decompose_padded_async)."""
    import torch

    if not isinstance(A, torch.Tensor) or not A.is_cuda or A.dtype != torch.complex128:
        raise TypeError("A must be a CUDA complex128 tensor (no CPU fallback)")
    if A.dim() != 2 or A.shape[0] != A.shape[1] or A.stride(1) != 1:
        raise ValueError("A must be square with unit column stride")
    m, lda = A.shape[0], A.stride(0)
    s = _structure(structure)
    if m == 0:  # the ABI rejects an empty matrix (EINVAL)
        _check(lib().ptdr_decompose_padded_async(None, 0, 0, s, None, None, 0, _stream_ptr(stream)),
               "ptdr_decompose_padded_async")
    n = max(1, (m - 1).bit_length())
    out = _out(out, 4 ** n, A.device, stream)
    nb = int(lib().ptdr_padded_workspace_bytes(m, s))
    if nb == ctypes.c_size_t(-1).value:
        raise PtdrError(PTDR_EINVAL, f"invalid (m={m}, structure={structure})")
    if workspace is None:
        workspace = torch.empty(max(nb, 1), dtype=torch.uint8, device=A.device)
        _keep_for_stream(stream, workspace)
    elif workspace.device != A.device:
        raise ValueError("workspace must be on A's device")
    _check(lib().ptdr_decompose_padded_async(ctypes.c_void_p(A.data_ptr()), m, lda, s,
                                             ctypes.c_void_p(out.data_ptr()),
                                             ctypes.c_void_p(workspace.data_ptr()), workspace.numel(),
                                             _stream_ptr(stream)), "ptdr_decompose_padded_async")
    return out


def decompose_generated(n: int, seed: int, rank: int = 0, world: int = 1, out=None, workspace=None,
                        stream=None, device=None):
    """Matrix-free decomposition of the seeded GENERAL matrix (ptdr_decompose_generated_async):
    the entries are computed inside the kernel, A is never stored."""
    import torch

    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    out = _out(out, (1 << (2 * n)) // world, dev, stream)
    nb = int(lib().ptdr_generated_workspace_bytes(n, world))
    if nb == ctypes.c_size_t(-1).value:
        raise PtdrError(PTDR_EINVAL, f"invalid (n={n}, world={world})")
    if workspace is None:
        workspace = torch.empty(max(nb, 1), dtype=torch.uint8, device=dev)
        _keep_for_stream(stream, workspace)
    else:
        _require_workspace(workspace, nb, dev)
    _check(lib().ptdr_decompose_generated_async(n, seed, rank, world, ctypes.c_void_p(out.data_ptr()),
                                                ctypes.c_void_p(workspace.data_ptr()), workspace.numel(),
                                                _stream_ptr(stream)), "ptdr_decompose_generated_async")
    return out


def decompose_peer(shard_ptrs, n: int, rank: int, world: int, out=None, workspace=None, stream=None,
                   device=None):
    """Per-rank decomposition reading every rank's row-block shard directly (TMA over
    NVLink; ptdr_decompose_peer_async).  shard_ptrs: device addresses (ints) of the
    `world` shards, in rank order, all readable from this GPU."""
    import torch

    if len(shard_ptrs) != world:
        raise ValueError("one shard pointer per rank")
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    out = _out(out, (1 << (2 * n)) // world, dev, stream)
    workspace = _workspace(workspace, n, "general", world, dev, stream)
    arr = (ctypes.c_void_p * world)(*[ctypes.c_void_p(int(p)) for p in shard_ptrs])
    _check(lib().ptdr_decompose_peer_async(arr, n, rank, world, ctypes.c_void_p(out.data_ptr()),
                                           ctypes.c_void_p(workspace.data_ptr()), workspace.numel(),
                                           _stream_ptr(stream)), "ptdr_decompose_peer_async")
    return out


def ipc_handle(tensor):
    """(opaque CUDA IPC handle of the allocation holding `tensor`, byte offset of the tensor)."""
    size = int(lib().ptdr_ipc_handle_size())
    buf = ctypes.create_string_buffer(size)
    off = ctypes.c_uint64()
    _check(lib().ptdr_ipc_get_handle(ctypes.c_void_p(tensor.data_ptr()), buf, ctypes.byref(off)),
           "ptdr_ipc_get_handle")
    return buf.raw, int(off.value)


def ipc_open(handle: bytes) -> int:
    """Map a peer allocation; returns its base device address (add the peer's offset)."""
    p = ctypes.c_void_p()
    _check(lib().ptdr_ipc_open(ctypes.c_char_p(handle), ctypes.byref(p)), "ptdr_ipc_open")
    return int(p.value)


def ipc_close(ptr: int):
    _check(lib().ptdr_ipc_close(ctypes.c_void_p(ptr)), "ptdr_ipc_close")


def decompose_zshard(band, structure, rank: int, world: int, out=None, workspace=None, stream=None):
    """Per-rank z-slice of a DIAGONAL / TRIDIAGONAL decomposition (ptdr_decompose_zshard_async):
    every rank holds the whole band, rank r writes z in [r 2^n/world, (r+1) 2^n/world) of
    every output block (block-major, output_count / world elements)."""
    import torch

    _require_cuda_c128(band, "band")
    s = _structure(structure)
    n = n_of(band, s)
    if world < 1 or world & (world - 1) or world > (1 << n) or not 0 <= rank < world:
        raise ValueError(f"invalid rank {rank} / world {world}")
    out = _out(out, output_count(n, s) // world, band.device, stream)
    workspace = _workspace(workspace, n, s, world, band.device, stream)
    st = lib().ptdr_decompose_zshard_async(ctypes.c_void_p(band.data_ptr()), n, s, rank, world,
                                           ctypes.c_void_p(out.data_ptr()),
                                           ctypes.c_void_p(workspace.data_ptr()), workspace.numel(),
                                           _stream_ptr(stream))
    _check(st, "ptdr_decompose_zshard_async")
    return out


def band_xmasks(n: int, s: int):
    """Ascending X-masks of the (2s+1)-band support (block order of decompose_band)."""
    import numpy as np

    cnt = int(lib().ptdr_band_xmask_count(n, s))
    if cnt == 0:
        raise PtdrError(PTDR_EINVAL, f"invalid (n={n}, s={s})")
    xs = np.empty(cnt, dtype=np.uint64)
    _check(lib().ptdr_band_xmasks(n, s, xs.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), cnt),
           "ptdr_band_xmasks")
    return xs


def decompose_band(diags, s: int, out=None, workspace=None, stream=None):
    """(2s+1)-band matrix given as diags[2s+1][2^n] (diags[d+s][i] = A[i][i+d]) -> the
    [len(band_xmasks(n, s))][2^n] nonzero-X-mask coefficient blocks (ptdr_decompose_band_async)."""
    import torch

    _require_cuda_c128(diags, "diags")
    if diags.dim() != 2 or diags.shape[0] != 2 * s + 1:
        raise ValueError("diags must be [2s+1, 2^n]")
    N = diags.shape[1]
    n = N.bit_length() - 1
    if (1 << n) != N:
        raise ValueError("2^n columns")
    cnt = int(lib().ptdr_band_xmask_count(n, s))
    if cnt == 0:
        raise PtdrError(PTDR_EINVAL, f"invalid (n={n}, s={s})")
    out = _out(out, cnt * N, diags.device, stream)
    nb = int(lib().ptdr_band_workspace_bytes(n, s))
    if workspace is None:
        workspace = torch.empty(max(nb, 1), dtype=torch.uint8, device=diags.device)
        _keep_for_stream(stream, workspace)
    else:
        _require_workspace(workspace, nb, diags.device)
    st = lib().ptdr_decompose_band_async(ctypes.c_void_p(diags.data_ptr()), n, s, ctypes.c_void_p(out.data_ptr()),
                                         ctypes.c_void_p(workspace.data_ptr()), workspace.numel(),
                                         _stream_ptr(stream))
    _check(st, "ptdr_decompose_band_async")
    return out


def _n_of_coeffs(c) -> int:
    n = (c.numel().bit_length() - 1) // 2
    if 4 ** n != c.numel():
        raise ValueError("coefficient arrays hold 4^n elements")
    return n


def reconstruct(coeffs, out=None, workspace=None, stream=None):
    """Inverse transform A = sum_P alpha_P P (ptdr_reconstruct_async): [2^n, 2^n] complex128."""
    import torch

    _require_cuda_c128(coeffs, "coeffs")
    n = _n_of_coeffs(coeffs)
    if out is None:
        out = torch.empty((1 << n, 1 << n), dtype=torch.complex128, device=coeffs.device)
        _keep_for_stream(stream, out)
    _require_cuda_c128(out, "out", 4 ** n, coeffs.device)
    nb = int(lib().ptdr_reconstruct_workspace_bytes(n))
    if workspace is None:
        workspace = torch.empty(nb, dtype=torch.uint8, device=coeffs.device)
        _keep_for_stream(stream, workspace)
    else:
        _require_workspace(workspace, nb, coeffs.device)
    _check(lib().ptdr_reconstruct_async(ctypes.c_void_p(coeffs.data_ptr()), n, ctypes.c_void_p(out.data_ptr()),
                                        ctypes.c_void_p(workspace.data_ptr()), workspace.numel(),
                                        _stream_ptr(stream)), "ptdr_reconstruct_async")
    return out


def reconstruct_matrix_layout(M, out=None, workspace=None, stream=None, inplace=False):
    """Inverse transform from the matrix layout M[z][z ^ x] = alpha(x, z) (what
    decompose(..., inplace=True) / decompose_matrix_layout return) to the dense matrix
    (ptdr_reconstruct_matrix_layout_async).  inplace=True overwrites M with A."""
    import torch

    _require_cuda_c128(M, "M")
    n = _n_of_coeffs(M)
    if inplace:
        if out is not None:
            raise ValueError("inplace=True writes into M; out must be None")
        out = M
    elif out is None:
        out = torch.empty((1 << n, 1 << n), dtype=torch.complex128, device=M.device)
        _keep_for_stream(stream, out)
    _require_cuda_c128(out, "out", 4 ** n, M.device)
    nb = int(lib().ptdr_reconstruct_matrix_layout_workspace_bytes(n))
    if workspace is None:
        workspace = torch.empty(nb, dtype=torch.uint8, device=M.device)
        _keep_for_stream(stream, workspace)
    else:
        _require_workspace(workspace, nb, M.device)
    _check(lib().ptdr_reconstruct_matrix_layout_async(ctypes.c_void_p(M.data_ptr()), n,
                                                      ctypes.c_void_p(out.data_ptr()),
                                                      ctypes.c_void_p(workspace.data_ptr()),
                                                      workspace.numel() * workspace.element_size(),
                                                      _stream_ptr(stream)), "ptdr_reconstruct_matrix_layout_async")
    return out


def axpby(mu, x, nu, y, out=None, stream=None):
    """Coefficients of mu A + nu B from those of A (x) and B (y) (ptdr_axpby_async)."""
    import torch

    _require_cuda_c128(x, "x")
    _require_cuda_c128(y, "y", x.numel(), x.device)
    out = _out(out, x.numel(), x.device, stream)
    mu, nu = complex(mu), complex(nu)
    _check(lib().ptdr_axpby_async(ctypes.c_void_p(out.data_ptr()), mu.real, mu.imag, ctypes.c_void_p(x.data_ptr()),
                                  nu.real, nu.imag, ctypes.c_void_p(y.data_ptr()), x.numel(), _stream_ptr(stream)),
           "ptdr_axpby_async")
    return out


def block_diag(blocks, out=None, stream=None):
    """Coefficients of diag(A_0, ..., A_{2^k-1}) from blocks[2^k][4^n] (ptdr_block_diag_async)."""
    import torch

    _require_cuda_c128(blocks, "blocks")
    nb = blocks.shape[0]
    k = nb.bit_length() - 1
    if (1 << k) != nb or blocks.dim() != 2:
        raise ValueError("blocks must be [2^k, 4^n]")
    n = _n_of_coeffs(blocks[0])
    out = _out(out, 4 ** (n + k), blocks.device, stream)
    _check(lib().ptdr_block_diag_async(ctypes.c_void_p(blocks.data_ptr()), n, k, ctypes.c_void_p(out.data_ptr()),
                                       _stream_ptr(stream)), "ptdr_block_diag_async")
    return out


def direct_sum(a, b, out=None, stream=None):
    """Coefficients of A (+) B (l.537-540) = block_diag with k = 1."""
    import torch

    return block_diag(torch.stack([a, b]).contiguous(), out=out, stream=stream)


def hermitian_augment(coeffs, out=None, stream=None):
    """Coefficients of [[0, A^*], [A, 0]] (ptdr_hermitian_augment_async)."""
    import torch

    _require_cuda_c128(coeffs, "coeffs")
    n = _n_of_coeffs(coeffs)
    out = _out(out, 4 ** (n + 1), coeffs.device, stream)
    _check(lib().ptdr_hermitian_augment_async(ctypes.c_void_p(coeffs.data_ptr()), n, ctypes.c_void_p(out.data_ptr()),
                                              _stream_ptr(stream)), "ptdr_hermitian_augment_async")
    return out


_DENSE_VARIANTS = {"general": 0, "hermitian": 1, "real_symmetric": 2}


def fro2_partials(device=None):
    """A zeroed device array for the ||.||_F^2 partials of the generators / sumsq."""
    import torch

    return torch.zeros(int(lib().ptdr_fro2_partial_count()), dtype=torch.float64, device=device or "cuda")


def fro2_total(partials) -> float:
    """Sum of the partials (copied to the host, exactly rounded sum: math.fsum)."""
    import math

    return math.fsum(partials.cpu().tolist())


def sumsq(x, partials=None, stream=None) -> float:
    """sum |x_e|^2 of a CUDA complex128 tensor by ptdr_sumsq_async (Parseval's left side)."""
    _require_cuda_c128(x, "x")
    if partials is None:
        partials = fro2_partials(x.device)
        _keep_for_stream(stream, partials)
    _check(lib().ptdr_sumsq_async(ctypes.c_void_p(x.data_ptr()), x.numel(), ctypes.c_void_p(partials.data_ptr()),
                                  _stream_ptr(stream)), "ptdr_sumsq_async")
    return fro2_total(partials)


def _fro2_ptr(fro2):
    if fro2 is None:
        return None
    import torch

    if not isinstance(fro2, torch.Tensor) or fro2.dtype != torch.float64 or not fro2.is_cuda or \
            fro2.numel() < int(lib().ptdr_fro2_partial_count()):
        raise ValueError("fro2 must be a CUDA float64 tensor of ptdr_fro2_partial_count() elements")
    return ctypes.c_void_p(fro2.data_ptr())


def generate_dense(n: int, seed: int, variant="general", row0: int = 0, nrows=None, out=None,
                   device=None, stream=None, fro2=None):
    """Seeded dense input (row block [row0, row0 + nrows)); fro2 (optional, fro2_partials())
    receives the ||A||_F^2 partials of the written rows."""
    import torch

    v = _DENSE_VARIANTS.get(variant, variant)
    N = 1 << n
    nrows = N - row0 if nrows is None else nrows
    if out is None:
        out = torch.empty((nrows, N), dtype=torch.complex128, device=device or "cuda")
        _keep_for_stream(stream, out)
    _require_cuda_c128(out, "out", nrows * N)
    st = lib().ptdr_generate_dense_async(n, seed, int(v), row0, nrows,
                                         ctypes.c_void_p(out.data_ptr()), _fro2_ptr(fro2), _stream_ptr(stream))
    _check(st, "ptdr_generate_dense_async")
    return out


def generate_band(n: int, seed: int, variant="tridiagonal", out=None, device=None, stream=None, fro2=None):
    import torch

    v = _structure(variant)
    shape = (1 << n,) if v == 3 else (2, 1 << n) if v == 6 else (3, 1 << n)
    if out is None:
        out = torch.empty(shape, dtype=torch.complex128, device=device or "cuda")
        _keep_for_stream(stream, out)
    _require_cuda_c128(out, "out", shape[0] if v == 3 else shape[0] << n)
    st = lib().ptdr_generate_band_async(n, seed, v, ctypes.c_void_p(out.data_ptr()), _fro2_ptr(fro2),
                                        _stream_ptr(stream))
    _check(st, "ptdr_generate_band_async")
    return out


def generate_sendblocks(n: int, seed: int, rank: int, world: int, out=None, device=None,
                        stream=None, subranges: int = 1, fro2=None):
    """Rank `rank`'s row block in the all-to-all send layout [K][world][K][R/K][R/K]
    (K = subranges; include/ptdr.h ptdr_generate_sendblocks_async).  Returned as
    [K, world, R/K * R] so that slice s is the contiguous equal-split send buffer of
    sub-range s (K = 1: [1, world, R * R])."""
    import torch

    N = 1 << n
    R = N // world
    K = subranges
    if out is None:
        out = torch.empty((K, world, R * R // K), dtype=torch.complex128, device=device or "cuda")
        _keep_for_stream(stream, out)
    _require_cuda_c128(out, "out", world * R * R)
    st = lib().ptdr_generate_sendblocks_async(n, seed, rank, world, K,
                                              ctypes.c_void_p(out.data_ptr()), _fro2_ptr(fro2),
                                              _stream_ptr(stream))
    _check(st, "ptdr_generate_sendblocks_async")
    return out


# ---- index helpers (host-side bookkeeping of the q order, include/ptdr.h) ----------
def q_of(x: int, z: int, n: int) -> int:
    """q index of the string with X-mask x and Z-mask z (code = 2 z_l + (x_l ^ z_l))."""
    q = 0
    for l in range(n):
        xl, zl = (x >> l) & 1, (z >> l) & 1
        q |= (2 * zl + (xl ^ zl)) << (2 * l)
    return q


def matrix_index(x: int, z: int, n: int):
    """(row, column) of coefficient (x, z) in the in-place matrix layout: (z, z ^ x)."""
    return z, z ^ x


def q_to_matrix_flat(q, n: int):
    """Flat index z * 2^n + (z ^ x) of the in-place layout for q indices (numpy, vectorised)."""
    import numpy as np

    q = np.asarray(q, dtype=np.int64)
    x = np.zeros_like(q)
    z = np.zeros_like(q)
    for l in range(n):
        c = (q >> (2 * l)) & 3
        zl = c >> 1
        x |= ((c & 1) ^ zl) << l
        z |= zl << l
    return (z << n) | (z ^ x)


def xz_of(q: int, n: int):
    x = z = 0
    for l in range(n):
        c = (q >> (2 * l)) & 3
        zl = c >> 1
        xl = (c & 1) ^ zl
        x |= xl << l
        z |= zl << l
    return x, z
