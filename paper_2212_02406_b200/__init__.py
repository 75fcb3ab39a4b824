"""B200-native Nested Neumann hot path (arXiv 2212.02406) — Python mirror.

This module binds ``libnnb.so`` (the C-ABI in ``include/nnb.h``) with ctypes
and mirrors the reference's C++ API (``/root/reference/proj/include/nn``):
same function names, same argument meaning, same error classes.  Arrays may
be numpy (host) or CUDA torch tensors (device); ``complex128`` inputs take the
``_z`` entry points, everything else is float64.  There is no CPU fallback —
importing works anywhere, but every compute call needs the CUDA library and a
GPU and raises otherwise.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from pathlib import Path
from typing import Optional

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libnnb.so"

# --------------------------------------------------------------------- errors
# Mirrors proj/include/nn/errors.hpp:10-71.


class Error(RuntimeError):
    pass


class ShapeError(Error):
    pass


class DomainError(Error):
    pass


class DivergenceError(Error):
    def __init__(self, msg: str, nest_index: int):
        super().__init__(msg)
        self.nest_index = nest_index


class ContractionError(Error):
    pass


class PlanError(Error):
    pass


class BudgetError(Error):
    pass


class DeviceError(Error):
    """CUDA / NCCL / OOM / no device (the library has no CPU fallback)."""


class SingularMatrixError(Error):
    def __init__(self, msg: str, pivot_index: int):
        super().__init__(msg)
        self.pivot_index = pivot_index


_STATUS = {1: ShapeError, 2: DomainError, 3: DivergenceError, 4: ContractionError, 5: PlanError,
           6: BudgetError, 7: DeviceError, 8: DeviceError, 9: DeviceError, 10: DeviceError, 11: SingularMatrixError}

ORDER_NORTHSTAR, ORDER_REFERENCE, ORDER_SYMMETRIC = 0, 1, 2
X0_GIVEN, X0_SCALED_IDENTITY, X0_TRANSPOSE_NORM, X0_JACOBI = 0, 1, 2, 3


class ChainConfig(C.Structure):
    _fields_ = [("depth_p", C.c_int32), ("max_iters", C.c_int32), ("tol", C.c_double),
                ("order", C.c_int32), ("x0_kind", C.c_int32), ("x0_scale", C.c_double),
                ("final_residual", C.c_int32)]


class ChainResult(C.Structure):
    _fields_ = [("iters", C.c_int32), ("fail_iter", C.c_int32), ("stopped", C.c_int32),
                ("products", C.c_int32), ("last_eps", C.c_double), ("device_ms", C.c_double)]


_dp = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int32
_SIGS = {
    "nnb_abi_version": ([], C.c_int),
    "nnb_last_error": ([], C.c_char_p),
    "nnb_device_count": ([], C.c_int),
    "nnb_kernel_launches": ([], C.c_uint64),
    "nnb_release_cached_memory": ([], C.c_int),
    "nnb_set_arithmetic": ([_i32], C.c_int),
    "nnb_get_arithmetic": ([], C.c_int32),
    "nnb_ozaki_moduli": ([_i64], C.c_int32),
    "nnb_chain_capture_residual": ([C.c_void_p, _i64], C.c_int),
    "nnb_ozaki_profile": ([_i32], None),
    "nnb_ozaki_stats": ([C.c_void_p, C.c_void_p, C.c_void_p, _i32], None),
    "nnb_gemm_d": ([_dp, _i64, _dp, _i64, _dp, _i64, _i64, _i64, _i64, _dp], C.c_int),
    "nnb_gemm_z": ([_dp, _dp, _dp, _i64, _i64, _i64, _dp], C.c_int),
    "nnb_gemm_nt_d": ([_dp, _i64, _dp, _i64, _dp, _i64, _i64, _i64, _i64, _dp], C.c_int),
    "nnb_axpby_d": ([C.c_double, _dp, C.c_double, _dp, C.c_double, _dp, _i64, _i64, _dp], C.c_int),
    "nnb_axpby_z": ([_dp, _dp, _dp, _dp, _dp, _dp, _i64, _i64, _dp], C.c_int),
    "nnb_frobenius_d": ([_dp, _i64, _dp, _dp], C.c_int),
    "nnb_frobenius_z": ([_dp, _i64, _dp, _dp], C.c_int),
    "nnb_trace_z": ([_dp, _i64, _dp, _dp], C.c_int),
    "nnb_residual_eps_d": ([_dp, _dp, _i64, _dp, _dp], C.c_int),
    "nnb_residual_eps_z": ([_dp, _dp, _i64, _dp, _dp], C.c_int),
    "nnb_x0_d": ([_dp, _i64, _i32, C.c_double, _dp, _dp], C.c_int),
    "nnb_nn_chain_d": ([_dp, _i64, _dp, C.POINTER(ChainConfig), _dp, _dp, C.POINTER(ChainResult), _dp],
                       C.c_int),
    "nnb_nn_chain_z": ([_dp, _i64, _dp, C.POINTER(ChainConfig), _dp, _dp, C.POINTER(ChainResult), _dp],
                       C.c_int),
    "nnb_nn_step_d": ([_dp, _dp, _i64, _i32, _dp, _dp], C.c_int),
    "nnb_nn_step_z": ([_dp, _dp, _i64, _i32, _dp, _dp], C.c_int),
    "nnb_ns_sum_d": ([_dp, _dp, _i64, _i64, _dp, _dp, _dp], C.c_int),
    "nnb_ns_sum_z": ([_dp, _dp, _i64, _i64, _dp, _dp, _dp], C.c_int),
    "nnb_nn_batched_z": ([_dp, _i64, _i32, _i32, _i32, _dp, _dp, _dp], C.c_int),
    "nnb_ns_batched_z": ([_dp, _i64, _i32, _i32, _dp, _dp], C.c_int),
    "nnb_ns_factorized_d": ([_dp, _dp, _i64, _i64, _dp, _dp, _dp], C.c_int),
    "nnb_ns_factorized_z": ([_dp, _dp, _i64, _i64, _dp, _dp, _dp], C.c_int),
    "nnb_power_ladder_d": ([_dp, _i64, C.c_uint64, _dp, _dp, _dp], C.c_int),
    "nnb_power_ladder_z": ([_dp, _i64, C.c_uint64, _dp, _dp, _dp], C.c_int),
    "nnb_nn_explicit_d": ([_dp, _dp, _i64, _i64, _i64, _dp, _dp, _dp], C.c_int),
    "nnb_nn_explicit_z": ([_dp, _dp, _i64, _i64, _i64, _dp, _dp, _dp], C.c_int),
    "nnb_mimo_detect_z": ([_dp, _dp, _i64, _i32, _i32, C.c_double, _i32, _i32, _dp, _dp, _dp, _dp], C.c_int),
    "nnb_spmv_block_d": ([_dp, _dp, _dp, _i64, _i64, _dp, _i64, _dp, _dp], C.c_int),
    "nnb_sparse_factorized_d": ([_dp, _dp, _dp, _i64, _i64, _dp, _i64, _i64, C.c_double, _dp, _dp, _dp,
                                 _dp], C.c_int),
    "nnb_sparse_last_bytes_per_nnz": ([], C.c_int),
    "nnb_sparse_last_matrix_bytes": ([], C.c_int64),
    "nnb_sparse_last_format": ([], C.c_char_p),
    "nnb_sparse_last_solve_ms": ([], C.c_double),
    "nnb_gaussian_stream": ([C.c_uint64, _i64, _dp], C.c_int),
    "nnb_householder_q_d": ([_dp, _i64, _dp, _dp], C.c_int),
    "nnb_householder_q_z": ([_dp, _i64, _dp, _dp], C.c_int),
    "nnb_random_spd_d": ([_dp, _dp, _i64, _dp, _dp], C.c_int),
    "nnb_random_conditioned_z": ([_dp, _dp, _dp, _i64, _dp, _dp], C.c_int),
    "nnb_direct_inverse_d": ([_dp, _i64, _dp, C.POINTER(C.c_int32), _dp], C.c_int),
    "nnb_direct_inverse_z": ([_dp, _i64, _dp, C.POINTER(C.c_int32), _dp], C.c_int),
    "nnb_transpose_d": ([_dp, _i64, _i64, _dp, _dp], C.c_int),
    "nnb_conj_transpose_z": ([_dp, _i64, _i64, _dp, _dp], C.c_int),
    "nnb_spectral_norm_z": ([_dp, _i64, _dp, C.c_double, _i32, _dp, _dp, _dp, _dp], C.c_int),
    "nnb_spectral_norm_shifted_csr": ([_dp, _dp, _dp, _i64, _i64, C.c_double, _dp, C.c_double, _i32, _dp, _dp,
                                       _dp, _dp], C.c_int),
    "nnb_partition_rows": ([_i64, _i32, _i32, C.POINTER(_i64), C.POINTER(_i64)], None),
    "nnb_comm_unique_id": ([_dp], C.c_int),
    "nnb_comm_init": ([_dp, _i32, _i32, C.POINTER(C.c_void_p)], C.c_int),
    "nnb_comm_destroy": ([C.c_void_p], C.c_int),
    "nnb_nn_chain_sharded_d": ([C.c_void_p, _dp, _i64, _dp, C.POINTER(ChainConfig), _dp, _dp,
                                C.POINTER(ChainResult), _dp], C.c_int),
    "nnb_nn_chain_sharded_emulated_d": ([_dp, _i64, _i32, _dp, C.POINTER(ChainConfig), _dp, _dp,
                                         C.POINTER(ChainResult), _dp], C.c_int),
    "nnb_sparse_factorized_sharded_d": ([C.c_void_p, _dp, _dp, _dp, _i64, _dp, _i64, _i64, C.c_double, _dp, _dp,
                                         _dp, _dp], C.c_int),
    "nnb_sparse_factorized_sharded_emulated_d": ([_dp, _dp, _dp, _i64, _i64, _dp, _i64, _i64, C.c_double, _i32,
                                                  _dp, _dp, _dp, _dp], C.c_int),
    "nnb_sparse_plan_create": ([C.c_void_p, _dp, _dp, _dp, _i64, _i64, C.POINTER(C.c_void_p), _dp], C.c_int),
    "nnb_sparse_plan_solve": ([C.c_void_p, _dp, _i64, C.c_double, _dp, _dp, _dp, _dp], C.c_int),
    "nnb_sparse_plan_destroy": ([C.c_void_p], C.c_int),
}

_lib: Optional[C.CDLL] = None


def lib() -> C.CDLL:
    """Load libnnb.so (fails loudly when the CUDA library was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise DeviceError(f"{LIB_PATH} is missing: build it with `make` (no CPU fallback exists)")
        L = C.CDLL(str(LIB_PATH))
        for name, (args, res) in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGS)


def release_cached_memory() -> None:
    """Return libnnb's cached work buffers (its stream-ordered pool) to the driver."""
    _check(lib().nnb_release_cached_memory())


def kernel_launches() -> int:
    return int(lib().nnb_kernel_launches())


ARITH_FAST, ARITH_REFERENCE, ARITH_OZAKI, ARITH_DMMA = 0, 1, 2, 3


class arithmetic:
    """Context manager: run real dense products in the given arithmetic mode of the
    calling thread (nnb_set_arithmetic), restoring the previous mode on exit."""

    def __init__(self, mode: int):
        self.mode = mode

    def __enter__(self):
        self._prev = lib().nnb_get_arithmetic()
        _check(lib().nnb_set_arithmetic(self.mode))
        return self

    def __exit__(self, *exc):
        lib().nnb_set_arithmetic(self._prev)


def ozaki_moduli(k: int) -> int:
    """Moduli the int8 emulation uses for inner dimension k (each is one int8 GEMM)."""
    return int(lib().nnb_ozaki_moduli(int(k)))


def ozaki_profile(on: bool) -> None:
    lib().nnb_ozaki_profile(1 if on else 0)


def ozaki_stats(reset: bool = True) -> dict:
    """Summed device time (CUDA events), work and launch count of the emulation's kernels
    recorded while ozaki_profile(True): classes gemm (int8 ops), split and recon (bytes)."""
    ms, work = (C.c_double * 3)(), (C.c_double * 3)()
    n = (C.c_int64 * 3)()
    lib().nnb_ozaki_stats(C.addressof(ms), C.addressof(work), C.addressof(n), 1 if reset else 0)
    return {name: {"ms": ms[i], "work": work[i], "launches": n[i]}
            for i, name in enumerate(("gemm", "split", "recon"))}


class reference_arithmetic(arithmetic):
    """Reference-exact mode (bit-identical to the reference; CUDA-core FP64, a
    verification mode)."""

    def __init__(self):
        super().__init__(ARITH_REFERENCE)


class dmma_arithmetic(arithmetic):
    """Every product on the FP64 tensor pipe (DMMA), no int8 emulation."""

    def __init__(self):
        super().__init__(ARITH_DMMA)


class ozaki_arithmetic(arithmetic):
    """Real products emulated on the int8 tensor cores (Ozaki scheme II, csrc/ozaki.cu)."""

    def __init__(self):
        super().__init__(ARITH_OZAKI)


def _check(status: int, index: int = 0) -> None:
    if status == 0:
        return
    msg = lib().nnb_last_error().decode(errors="replace")
    cls = _STATUS.get(status, Error)
    if cls in (DivergenceError, SingularMatrixError):
        raise cls(msg, index)
    raise cls(msg)


# ---------------------------------------------------------------- array glue
def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


def _ptr(a) -> int:
    if a is None:
        return None
    if _is_torch(a):
        return a.data_ptr()
    return a.ctypes.data


def _prep(a, complex_: bool):
    """Contiguous float64/complex128 array, keeping torch CUDA tensors on device."""
    if _is_torch(a):
        import torch

        dt = torch.complex128 if complex_ else torch.float64
        return a.to(dt).contiguous()
    return np.ascontiguousarray(np.asarray(a), dtype=np.complex128 if complex_ else np.float64)


def _is_complex(*arrs) -> bool:
    for a in arrs:
        if a is None:
            continue
        if _is_torch(a):
            if a.is_complex():
                return True
        elif np.iscomplexobj(a):
            return True
    return False


def _empty_like(a, shape=None):
    shape = tuple(a.shape) if shape is None else shape
    if _is_torch(a):
        import torch

        return torch.empty(shape, dtype=a.dtype, device=a.device)
    return np.empty(shape, dtype=a.dtype)


def _stream(a) -> Optional[int]:
    if _is_torch(a) and a.is_cuda:
        import torch

        return torch.cuda.current_stream(a.device).cuda_stream
    return None


# ------------------------------------------------------------ kernels (L1)
def matmul(a, b):
    """nn::matmul (proj/include/nn/kernels.hpp:20-21) on the FP64 DMMA GEMM."""
    if a.shape[1] != b.shape[0]:
        raise ShapeError(f"matmul: inner dimensions disagree ({a.shape[1]} vs {b.shape[0]})")
    z = _is_complex(a, b)
    a, b = _prep(a, z), _prep(b, z)
    m, k = a.shape
    n = b.shape[1]
    out = _empty_like(a, (m, n))
    if z:
        _check(lib().nnb_gemm_z(_ptr(a), _ptr(b), _ptr(out), m, k, n, _stream(a)))
    else:
        _check(lib().nnb_gemm_d(_ptr(a), k, _ptr(b), n, _ptr(out), n, m, k, n, _stream(a)))
    return out


def matmul_nt(a, bt):
    """C = A·Bᵀ for real A (m×k) and Bᵀ (n×k): the K-major GEMM (also B·Bᵀ without a transpose)."""
    if a.shape[1] != bt.shape[1]:
        raise ShapeError("matmul_nt: inner dimensions disagree")
    a, bt = _prep(a, False), _prep(bt, False)
    m, k = a.shape
    n = bt.shape[0]
    out = _empty_like(a, (m, n))
    _check(lib().nnb_gemm_nt_d(_ptr(a), k, _ptr(bt), k, _ptr(out), n, m, k, n, _stream(a)))
    return out


def _axpby(alpha, a, beta=0.0, b=None, gamma=0.0):
    z = _is_complex(a, b) or any(isinstance(v, complex) and v.imag != 0 for v in (alpha, beta, gamma))
    a = _prep(a, z)
    b = _prep(b, z) if b is not None else None
    out = _empty_like(a)
    rows, cols = a.shape
    if z:
        co = lambda v: np.array([complex(v).real, complex(v).imag])
        al, be, ga = co(alpha), co(beta), co(gamma)
        _check(lib().nnb_axpby_z(al.ctypes.data, _ptr(a), be.ctypes.data, _ptr(b), ga.ctypes.data, _ptr(out),
                                 rows, cols, _stream(a)))
    else:
        _check(lib().nnb_axpby_d(float(alpha), _ptr(a), float(beta), _ptr(b), float(gamma), _ptr(out), rows, cols,
                                 _stream(a)))
    return out


def add(a, b):
    if a.shape != b.shape:
        raise ShapeError("add: shape mismatch")
    return _axpby(1.0, a, 1.0, b)


def sub(a, b):
    if a.shape != b.shape:
        raise ShapeError("sub: shape mismatch")
    return _axpby(1.0, a, -1.0, b)


def scale(m, factor):
    return _axpby(factor, m)


def identity_minus(m):
    if m.shape[0] != m.shape[1]:
        raise ShapeError("identity_minus: matrix must be square")
    return _axpby(-1.0, m, 0.0, None, 1.0)


def plus_identity(m):
    if m.shape[0] != m.shape[1]:
        raise ShapeError("plus_identity: matrix must be square")
    return _axpby(1.0, m, 0.0, None, 1.0)


def conjugate_transpose(a):
    """nn::conjugate_transpose (proj/include/nn/kernels.hpp:37): Aᵀ for real, Aᴴ for complex, on the device."""
    z = _is_complex(a)
    a = _prep(a, z)
    out = _empty_like(a, (a.shape[1], a.shape[0]))
    f = lib().nnb_conj_transpose_z if z else lib().nnb_transpose_d
    _check(f(_ptr(a), a.shape[0], a.shape[1], _ptr(out), _stream(a)))
    return out


def direct_inverse_oracle(a):
    """nn::direct_inverse_oracle (kernels.hpp:67): Gauss–Jordan with partial pivoting on the
    device, bit-identical to the reference for real input; SingularMatrixError(pivot_index)."""
    if a.shape[0] != a.shape[1]:
        raise ShapeError("direct_inverse_oracle: matrix must be square")
    z = _is_complex(a)
    a = _prep(a, z)
    out = _empty_like(a)
    piv = C.c_int32(-1)
    f = lib().nnb_direct_inverse_z if z else lib().nnb_direct_inverse_d
    _check(f(_ptr(a), a.shape[0], _ptr(out), C.byref(piv), _stream(a)), piv.value)
    return out


def frobenius_norm(m) -> float:
    z = _is_complex(m)
    m = _prep(m, z)
    out = C.c_double()
    f = lib().nnb_frobenius_z if z else lib().nnb_frobenius_d
    _check(f(_ptr(m), int(np.prod(m.shape)), C.addressof(out), _stream(m)))
    return out.value


def trace(m) -> complex:
    if m.shape[0] != m.shape[1]:
        raise ShapeError("trace: matrix must be square")
    m = _prep(m, True)
    out = np.zeros(2)
    _check(lib().nnb_trace_z(_ptr(m), m.shape[0], out.ctypes.data, _stream(m)))
    return complex(out[0], out[1])


def spmv_block(csr: "Csr", x):
    """nn::spmv_block (proj/include/nn/kernels.hpp:91-92): Y = W·X, X n×k."""
    if csr.n != x.shape[0]:
        raise ShapeError("spmv_block: inner dimensions disagree")
    x = _prep(x, False)
    y = _empty_like(x)
    k = 1 if x.ndim == 1 else x.shape[1]
    _check(lib().nnb_spmv_block_d(_ptr(csr.row_ptr), _ptr(csr.col), _ptr(csr.val), csr.n, csr.nnz, _ptr(x), k,
                                  _ptr(y), _stream(x)))
    return y


# ------------------------------------------------------------ solver (L3)
def residual_epsilon(phi, w_tilde) -> float:
    """eps = ||I − phi·W~||_F / sqrt(N) (proj/include/nn/solver.hpp:55)."""
    z = _is_complex(phi, w_tilde)
    phi, w = _prep(phi, z), _prep(w_tilde, z)
    out = C.c_double()
    f = lib().nnb_residual_eps_z if z else lib().nnb_residual_eps_d
    _check(f(_ptr(phi), _ptr(w), w.shape[0], C.addressof(out), _stream(w)))
    return out.value


def _square_conform(phi, w, who):
    if w.shape[0] != w.shape[1] or phi.shape != w.shape:
        raise ShapeError(f"{who}: shapes do not conform")


def nn_step(phi, w_tilde, depth_L: int):
    """One nest, exactly L+1 products (proj/include/nn/solver.hpp:68-69)."""
    _square_conform(phi, w_tilde, "nn_step")
    z = _is_complex(phi, w_tilde)
    phi, w = _prep(phi, z), _prep(w_tilde, z)
    out = _empty_like(phi)
    f = lib().nnb_nn_step_z if z else lib().nnb_nn_step_d
    _check(f(_ptr(phi), _ptr(w), w.shape[0], int(depth_L), _ptr(out), _stream(w)))
    return out


def newton_step(z_, w_tilde):
    """Z(2I − W~Z) ≡ nn_step(L=1) (proj/include/nn/solver.hpp:72-73)."""
    return nn_step(z_, w_tilde, 1)


def chebyshev_step(z_, w_tilde):
    """Z[3I − W~Z(3I − W~Z)] ≡ nn_step(L=2) (proj/include/nn/solver.hpp:76-77)."""
    return nn_step(z_, w_tilde, 2)


def ns_sum(phi0, w_tilde, order: int):
    """Truncated Neumann series (proj/include/nn/solver.hpp:61-62). Returns (sum, products)."""
    _square_conform(phi0, w_tilde, "ns_sum")
    z = _is_complex(phi0, w_tilde)
    phi0, w = _prep(phi0, z), _prep(w_tilde, z)
    out = _empty_like(phi0)
    prods = C.c_double()
    f = lib().nnb_ns_sum_z if z else lib().nnb_ns_sum_d
    _check(f(_ptr(phi0), _ptr(w), w.shape[0], int(order), _ptr(out), C.addressof(prods), _stream(w)))
    return out, prods.value


def ns_factorized(phi0, w_tilde, gamma: int):
    """Factorized Neumann series of order gamma = 2^s-1 (proj/src/factorized.cpp:42-61). Returns (sum, products)."""
    _square_conform(phi0, w_tilde, "ns_factorized")
    z = _is_complex(phi0, w_tilde)
    phi0, w = _prep(phi0, z), _prep(w_tilde, z)
    out = _empty_like(phi0)
    prods = C.c_double()
    f = lib().nnb_ns_factorized_z if z else lib().nnb_ns_factorized_d
    _check(f(_ptr(phi0), _ptr(w), w.shape[0], int(gamma), _ptr(out), C.addressof(prods), _stream(w)))
    return out, prods.value


def power_ladder(p, exponent: int):
    """p^exponent by square-and-multiply (proj/src/kernels.cpp:434-452). Returns (power, products)."""
    if p.shape[0] != p.shape[1]:
        raise ShapeError("power_ladder: matrix must be square")
    z = _is_complex(p)
    p = _prep(p, z)
    out = _empty_like(p)
    prods = C.c_double()
    f = lib().nnb_power_ladder_z if z else lib().nnb_power_ladder_d
    _check(f(_ptr(p), p.shape[0], int(exponent), _ptr(out), C.addressof(prods), _stream(p)))
    return out, prods.value


def nn_explicit(phi0, w_tilde, nests_i: int, depth_L: int):
    """Non-recursive product form of nests_i+1 nests of depth L (proj/src/solver.cpp:176-199)."""
    _square_conform(phi0, w_tilde, "nn_explicit")
    z = _is_complex(phi0, w_tilde)
    phi0, w = _prep(phi0, z), _prep(w_tilde, z)
    out = _empty_like(phi0)
    prods = C.c_double()
    f = lib().nnb_nn_explicit_z if z else lib().nnb_nn_explicit_d
    _check(f(_ptr(phi0), _ptr(w), w.shape[0], int(nests_i), int(depth_L), _ptr(out), C.addressof(prods), _stream(w)))
    return out, prods.value


def equivalent_ns_order(nests_i: int, depth_L: int) -> int:
    """(L+1)^(i+1) − 1 (proj/src/solver.cpp:201-205), exact (Python int)."""
    return (depth_L + 1) ** (nests_i + 1) - 1


@dataclass
class ChainReport:
    """Result of nn_chain: the reference's ConvergenceReport subset."""
    history: list
    iters: int
    stopped_reason: str
    products: int
    device_ms: float
    fail_iter: int = 0
    n3_multiplies: float = 0.0
    n2_ops: int = 0


def nn_chain(a, x0=None, *, p: int, max_iters: int, tol: float = 0.0, order: int = ORDER_NORTHSTAR,
             x0_kind: Optional[int] = None, x0_scale: float = 1.0, final_residual: bool = True, out=None,
             residual_out=None):
    """Nested Neumann chain from X0; returns (X, ChainReport).

    eps is recorded before every nest and after the last one; stops when
    eps < tol (tol > 0) or after max_iters nests.  residual_out (a device n×n float64
    tensor, real chains) receives the chain's own final residual R = I − A·X.
    """
    if residual_out is not None:
        _check(lib().nnb_chain_capture_residual(_ptr(residual_out), residual_out.shape[1]))
    n = a.shape[0]
    if a.shape != (n, n):
        raise ShapeError("nn chain: matrix must be square")
    z = _is_complex(a, x0)
    a = _prep(a, z)
    if x0_kind is None:
        x0_kind = X0_GIVEN if x0 is not None else X0_TRANSPOSE_NORM
    x0p = _prep(x0, z) if x0 is not None else None
    out = _empty_like(a) if out is None else out
    hist = np.zeros(max_iters + 1)
    cfg = ChainConfig(p, max_iters, tol, order, x0_kind, x0_scale, int(final_residual))
    res = ChainResult()
    f = lib().nnb_nn_chain_z if z else lib().nnb_nn_chain_d
    st = f(_ptr(a), n, _ptr(x0p), C.byref(cfg), _ptr(out), hist.ctypes.data, C.byref(res), _stream(a))
    _check(st, res.fail_iter)
    recorded = res.iters + (1 if final_residual or res.stopped == 0 else 0)
    rep = ChainReport(history=[(k, float(hist[k])) for k in range(recorded)], iters=res.iters,
                      stopped_reason="tolerance" if res.stopped == 0 else "max_nests", products=res.products,
                      device_ms=res.device_ms, n3_multiplies=float(res.iters * (p + 1)),
                      n2_ops=res.iters * (p + 1))
    return out, rep


@dataclass
class Normalization:
    """proj/include/nn/normalization.hpp:16-22."""
    theta: float = 0.0
    kind: str = "trace"
    k_order: int = 0
    contraction_norm: float = 0.0
    valid: bool = False


def normalize(w, norm: Normalization):
    """W~ = theta·W; ContractionError for an invalid normalization (normalization.cpp:94-99)."""
    if not norm.valid:
        raise ContractionError("normalize: normalization does not satisfy the contraction condition")
    return scale(w, norm.theta)


def nn_invert(w, norm: Normalization, depth_L: int = 2, max_nests: int = 64, tol: float = 1e-10):
    """nn::nn_invert (proj/src/solver.cpp:123-174): phi0 = I on W~ = theta·W,
    nests until eps < tol or the budget runs out; returns (theta·phi, report)."""
    if w.shape[0] != w.shape[1]:
        raise ShapeError("nn_invert: matrix must be square")
    if tol < 1e-15:
        raise DomainError("SolverConfig: tol below double precision (minimum 1e-15)")
    if max_nests < 1:
        raise DomainError("SolverConfig: max_nests must be >= 1")
    wt = normalize(w, norm)
    try:
        phi, rep = nn_chain(wt, None, p=depth_L, max_iters=max_nests, tol=tol, order=ORDER_REFERENCE,
                            x0_kind=X0_SCALED_IDENTITY, x0_scale=1.0)
    except DivergenceError as e:
        raise DivergenceError(f"nn_invert: non-finite iterate at nest {e.nest_index}", e.nest_index) from None
    rep.n3_multiplies = float(rep.iters * (depth_L + 1))
    rep.n2_ops = rep.iters * (depth_L + 1)  # captured before the final scale (solver.cpp:161-165)
    return scale(phi, norm.theta), rep


def x0(a, kind: int = X0_TRANSPOSE_NORM, scale_: float = 1.0):
    """Initial iterate builders (A^T/(||A||_1||A||_inf), diag(A)^-1, s·I)."""
    a = _prep(a, False)
    out = _empty_like(a)
    _check(lib().nnb_x0_d(_ptr(a), a.shape[0], kind, scale_, _ptr(out), _stream(a)))
    return out


# ------------------------------------------------------------ generators (§8(a) A14)
def gaussian_stream(seed: int, count: int) -> np.ndarray:
    """`count` draws of nn::GaussianStream(seed) (proj/include/nn/rng.hpp:15-52)."""
    out = np.empty(count)
    _check(lib().nnb_gaussian_stream(seed, count, out.ctypes.data if count else None))
    return out


def log_uniform_spectrum(n: int, cond: float) -> np.ndarray:
    """cond^-(n-1-j)/(n-1), j = 0..n-1, through C pow like the reference (kernels.cpp:116-124)."""
    if n == 1:
        return np.ones(1)
    return np.array([cond ** (-((n - 1 - j) / (n - 1))) for j in range(n)])


def householder_q(a):
    """Unitary factor of the Householder QR (kernels.cpp:64-105), on the device."""
    z = _is_complex(a)
    a = _prep(a, z)
    if a.shape[0] != a.shape[1]:
        raise ShapeError("householder_q: matrix must be square")
    out = _empty_like(a)
    f = lib().nnb_householder_q_z if z else lib().nnb_householder_q_d
    _check(f(_ptr(a), a.shape[0], _ptr(out), _stream(a)))
    return out


def random_spd(n: int, cond: float, seed: int) -> np.ndarray:
    """nn::random_spd (kernels.cpp:352-381), bit-identical: Q·diag(λ)·Qᵀ with Q from the
    Householder QR of a GaussianStream(seed) matrix, QR and products on the device."""
    if n < 1:
        raise DomainError("random_spd: n must be >= 1")
    if cond < 1.0:
        raise DomainError("random_spd: cond must be >= 1")
    g = gaussian_stream(seed, n * n).reshape(n, n)
    lam = log_uniform_spectrum(n, cond)
    out = np.empty((n, n))
    _check(lib().nnb_random_spd_d(g.ctypes.data, lam.ctypes.data, n, out.ctypes.data, None))
    return out


def random_conditioned_complex(n: int, cond: float, seed: int) -> np.ndarray:
    """nn::random_conditioned_complex (kernels.cpp:383-407): U·diag(σ)·Vᴴ, U and V the
    Householder Q of two complex GaussianStream(seed) draws (equal to a few ulps)."""
    if n < 1:
        raise DomainError("random_conditioned_complex: n must be >= 1")
    if cond < 1.0:
        raise DomainError("random_conditioned_complex: cond must be >= 1")
    g = gaussian_stream(seed, 4 * n * n)
    gu = np.ascontiguousarray(g[: 2 * n * n])
    gv = np.ascontiguousarray(g[2 * n * n:])
    sig = log_uniform_spectrum(n, cond)
    out = np.empty((n, n), np.complex128)
    _check(lib().nnb_random_conditioned_z(gu.ctypes.data, gv.ctypes.data, sig.ctypes.data, n, out.ctypes.data,
                                          None))
    return out


# ------------------------------------------------------------ multi-GPU (C4)
def partition_rows(n: int, world: int, rank: int) -> tuple[int, int]:
    """(row0, rows) of `rank`'s block in the sharded chain (16-row units, balanced)."""
    r0, rs = C.c_int64(), C.c_int64()
    lib().nnb_partition_rows(n, world, rank, C.byref(r0), C.byref(rs))
    return r0.value, rs.value


class Comm:
    """NCCL communicator owned by libnnb (one process per GPU)."""

    def __init__(self, world: int, rank: int, unique_id: bytes):
        self.world, self.rank = world, rank
        h = C.c_void_p()
        buf = C.create_string_buffer(bytes(unique_id), 128)
        _check(lib().nnb_comm_init(C.addressof(buf), world, rank, C.byref(h)))
        self.handle = h

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib().nnb_comm_unique_id(C.addressof(buf)))
        return buf.raw

    @classmethod
    def from_torch_distributed(cls):
        """Rank 0 creates the NCCL id, torch.distributed broadcasts it (plumbing only)."""
        import torch
        import torch.distributed as dist

        world, rank = dist.get_world_size(), dist.get_rank()
        t = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            t.copy_(torch.frombuffer(bytearray(cls.unique_id()), dtype=torch.uint8))
        dist.broadcast(t, 0)
        return cls(world, rank, bytes(t.cpu().numpy().tobytes()))

    def close(self):
        if self.handle:
            lib().nnb_comm_destroy(self.handle)
            self.handle = None


def _sharded_report(hist, res, p, final_residual):
    recorded = res.iters + (1 if final_residual or res.stopped == 0 else 0)
    return ChainReport(history=[(k, float(hist[k])) for k in range(recorded)], iters=res.iters,
                       stopped_reason="tolerance" if res.stopped == 0 else "max_nests", products=res.products,
                       device_ms=res.device_ms, fail_iter=res.fail_iter, n3_multiplies=float(res.iters * (p + 1)),
                       n2_ops=res.iters * (p + 1))


def nn_chain_sharded(comm: Comm, a_rows, n: int, x0_rows=None, *, p: int, max_iters: int, tol: float = 0.0,
                     x0_kind: Optional[int] = None, x0_scale: float = 1.0, final_residual: bool = True, out=None):
    """Row-sharded chain: this rank's rows of A in, its rows of X out."""
    a_rows = _prep(a_rows, False)
    if x0_kind is None:
        x0_kind = X0_GIVEN if x0_rows is not None else X0_TRANSPOSE_NORM
    x0p = _prep(x0_rows, False) if x0_rows is not None else None
    out = _empty_like(a_rows) if out is None else out
    hist = np.zeros(max_iters + 1)
    cfg = ChainConfig(p, max_iters, tol, ORDER_NORTHSTAR, x0_kind, x0_scale, int(final_residual))
    res = ChainResult()
    st = lib().nnb_nn_chain_sharded_d(comm.handle, _ptr(a_rows), n, _ptr(x0p), C.byref(cfg), _ptr(out),
                                      hist.ctypes.data, C.byref(res), _stream(a_rows))
    _check(st, res.fail_iter)
    return out, _sharded_report(hist, res, p, final_residual)


def nn_chain_sharded_emulated(a, world: int, x0=None, *, p: int, max_iters: int, tol: float = 0.0,
                              x0_kind: Optional[int] = None, x0_scale: float = 1.0, final_residual: bool = True):
    """The sharded schedule with `world` virtual ranks on this GPU (validation on one device)."""
    a = _prep(a, False)
    n = a.shape[0]
    if x0_kind is None:
        x0_kind = X0_GIVEN if x0 is not None else X0_TRANSPOSE_NORM
    x0p = _prep(x0, False) if x0 is not None else None
    out = _empty_like(a)
    hist = np.zeros(max_iters + 1)
    cfg = ChainConfig(p, max_iters, tol, ORDER_NORTHSTAR, x0_kind, x0_scale, int(final_residual))
    res = ChainResult()
    st = lib().nnb_nn_chain_sharded_emulated_d(_ptr(a), n, world, _ptr(x0p), C.byref(cfg), _ptr(out),
                                               hist.ctypes.data, C.byref(res), _stream(a))
    _check(st, res.fail_iter)
    return out, _sharded_report(hist, res, p, final_residual)


# ------------------------------------------------------------ batched (C2)
def nn_batched(a, p: int = 2, iters: int = 4, want_eps: bool = True, out=None):
    """Batched n×n complex NN inversion with Jacobi X0 (n = 16: batched_z16_kernel; n = 8, 24, 32:
    batched_generic.cu); returns (X, eps_last)."""
    a = _prep(a, True)
    b, n = a.shape[0], a.shape[1]
    out = _empty_like(a) if out is None else out
    eps = None
    if want_eps:
        if _is_torch(a):
            import torch

            eps = torch.empty(b, dtype=torch.float64, device=a.device)
        else:
            eps = np.empty(b)
    _check(lib().nnb_nn_batched_z(_ptr(a), b, n, p, iters, _ptr(out), _ptr(eps), _stream(a)))
    return out, eps


def mimo_detect(h, y, sigma2: float = 0.1, p: int = 2, iters: int = 4, want_x: bool = False,
                want_eps: bool = False):
    """Fused MIMO detection: A = HᴴH + σ²I, X = NN⁻¹(A), x̂ = X·Hᴴy per system.
    h: (batch, antennas, users) complex with users in {8, 16, 24, 32}, y: (batch, antennas) complex.
    Returns (x̂, X or None, eps or None)."""
    h = _prep(h, True)
    y = _prep(y, True)
    b, ant, users = h.shape
    xh = _empty_like(h, (b, users))
    x = _empty_like(h, (b, users, users)) if want_x else None
    eps = None
    if want_eps:
        if _is_torch(h):
            import torch

            eps = torch.empty(b, dtype=torch.float64, device=h.device)
        else:
            eps = np.empty(b)
    _check(lib().nnb_mimo_detect_z(_ptr(h), _ptr(y), b, ant, users, float(sigma2), p, iters, _ptr(xh), _ptr(x),
                                   _ptr(eps), _stream(h)))
    return xh, x, eps


def ns_batched(a, order: int):
    """Batched Neumann-series baseline (ns_sum of `order` terms from Jacobi X0)."""
    a = _prep(a, True)
    out = _empty_like(a)
    _check(lib().nnb_ns_batched_z(_ptr(a), a.shape[0], a.shape[1], order, _ptr(out), _stream(a)))
    return out


# ------------------------------------------------------------ sparse (C5)
@dataclass
class Csr:
    """CSR with int64 row_ptr, int32 col, float64 values (host numpy or device torch)."""
    row_ptr: object
    col: object
    val: object
    n: int
    nnz: int = field(default=0)

    def __post_init__(self):
        if not self.nnz:
            self.nnz = int(self.col.shape[0])


def solve_sparse_factorized(csr: Csr, b, gamma: int, norm: Normalization):
    """nn::solve_sparse_factorized (proj/src/factorized.cpp:101-140). Returns (x, spmv_count)."""
    if b.shape[0] != csr.n:
        raise ShapeError("solve_sparse_factorized: B row count does not match W")
    if not norm.valid:
        raise ContractionError("solve_sparse_factorized: invalid normalization")
    b = _prep(b, False)
    k = 1 if b.ndim == 1 else b.shape[1]
    out = _empty_like(b)
    cnt = C.c_int64()
    ff = C.c_int32(-1)
    st = lib().nnb_sparse_factorized_d(_ptr(csr.row_ptr), _ptr(csr.col), _ptr(csr.val), csr.n, csr.nnz, _ptr(b), k,
                                       int(gamma), float(norm.theta), _ptr(out), C.addressof(cnt), C.addressof(ff),
                                       _stream(b))
    _check(st, ff.value)
    return out, cnt.value


def sparse_last_bytes_per_nnz() -> int:
    """CSR bytes per nonzero the calling thread's last solve_sparse_factorized consumed:
    1 (pair dictionary), 10 (int16 column deltas) or 12 (int32 columns)."""
    return int(lib().nnb_sparse_last_bytes_per_nnz())


def sparse_last_matrix_bytes() -> int:
    """Operator bytes one application of the calling thread's last solve streamed."""
    return int(lib().nnb_sparse_last_matrix_bytes())


def sparse_last_format() -> str:
    """Name of the operator format the calling thread's last sparse solve consumed."""
    return lib().nnb_sparse_last_format().decode()


def sparse_last_solve_ms() -> float:
    """Device ms of the calling thread's last row-slab solve without its slab setup."""
    return float(lib().nnb_sparse_last_solve_ms())


def solve_sparse_factorized_sharded(comm: Comm, csr_rows: Csr, n: int, b_rows, gamma: int, norm: Normalization):
    """Row-slab sharded solve: this rank's CSR rows (global columns,
    row_ptr offsets into col/val), its rows of B in, its rows of x out."""
    if not norm.valid:
        raise ContractionError("solve_sparse_factorized: invalid normalization")
    b_rows = _prep(b_rows, False)
    k = 1 if b_rows.ndim == 1 else b_rows.shape[1]
    out = _empty_like(b_rows)
    cnt, ff = C.c_int64(), C.c_int32(-1)
    st = lib().nnb_sparse_factorized_sharded_d(comm.handle, _ptr(csr_rows.row_ptr), _ptr(csr_rows.col),
                                               _ptr(csr_rows.val), n, _ptr(b_rows), k, int(gamma),
                                               float(norm.theta), _ptr(out), C.addressof(cnt), C.addressof(ff),
                                               _stream(b_rows))
    _check(st, ff.value)
    return out, cnt.value


class SparseShardedPlan:
    """Prepared row slab for repeated sharded solves (nnb_sparse_plan_*)."""

    def __init__(self, comm: Comm, csr_rows: Csr, n: int, k: int = 1, stream_like=None):
        self.comm, self.n, self.k = comm, n, k
        self._keep = csr_rows  # the CSR arrays must outlive the plan when borrowed
        h = C.c_void_p()
        _check(lib().nnb_sparse_plan_create(comm.handle, _ptr(csr_rows.row_ptr), _ptr(csr_rows.col),
                                            _ptr(csr_rows.val), n, k, C.byref(h), _stream(stream_like)))
        self.handle = h

    def solve(self, b_rows, gamma: int, norm: Normalization):
        if not norm.valid:
            raise ContractionError("solve_sparse_factorized: invalid normalization")
        b_rows = _prep(b_rows, False)
        out = _empty_like(b_rows)
        cnt, ff = C.c_int64(), C.c_int32(-1)
        st = lib().nnb_sparse_plan_solve(self.handle, _ptr(b_rows), int(gamma), float(norm.theta), _ptr(out),
                                         C.addressof(cnt), C.addressof(ff), _stream(b_rows))
        _check(st, ff.value)
        return out, cnt.value

    def close(self):
        if self.handle:
            lib().nnb_sparse_plan_destroy(self.handle)
            self.handle = None


def solve_sparse_factorized_sharded_emulated(csr: Csr, b, gamma: int, norm: Normalization, world: int):
    """The row-slab schedule with `world` virtual ranks on this GPU."""
    if not norm.valid:
        raise ContractionError("solve_sparse_factorized: invalid normalization")
    b = _prep(b, False)
    k = 1 if b.ndim == 1 else b.shape[1]
    out = _empty_like(b)
    cnt, ff = C.c_int64(), C.c_int32(-1)
    st = lib().nnb_sparse_factorized_sharded_emulated_d(_ptr(csr.row_ptr), _ptr(csr.col), _ptr(csr.val), csr.n,
                                                        csr.nnz, _ptr(b), k, int(gamma), float(norm.theta), world,
                                                        _ptr(out), C.addressof(cnt), C.addressof(ff), _stream(b))
    _check(st, ff.value)
    return out, cnt.value


__all__ = [n for n in dir() if not n.startswith("_")]
