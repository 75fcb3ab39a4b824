"""ORACLE — test infrastructure only.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs
(``cpu_baseline`` and ``--impl reference``) may import this package, and only
as the checker / the reference CPU timing — never as the thing measured for
the GPU arm or shipped by the product (``paper_2212_02406_b200`` never imports
it).

Two checkers live here:

* ``ref``  — ``_ref/libnnref.so``: the UNMODIFIED reference sources
  (/root/reference/proj/src) compiled in place by ``oracle/Makefile`` with the
  ctypes harness ``ref_capi.cpp``.  Built in the dev container; travels to the
  GPU box as a prebuilt .so.
* ``port`` — ``lib/libnn_oracle.so``: the plain-C restatement ``nn_oracle.c``,
  pinned bit-for-bit against ``ref`` and against ``tests/golden/`` fixtures.

All matrices are numpy ``complex128`` row-major (the reference's
``std::complex<double>`` layout); real inputs are promoted.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SO = HERE / "_ref" / "libnnref.so"
PORT_SO = HERE / "lib" / "libnn_oracle.so"

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_ip = C.POINTER(C.c_int)


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str, index: int | None = None):
        super().__init__(f"status {status}: {msg}")
        self.status = status
        self.index = index


def _z(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128))


def _ptr(a: np.ndarray, t=_dp):
    return a.ctypes.data_as(t)


def build() -> None:
    """Compile the C restatement, and the reference harness when /root/reference exists."""
    import subprocess

    targets = ["lib/libnn_oracle.so"]
    if Path(os.environ.get("REF", "/root/reference"), "proj", "src", "solver.cpp").exists():
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", str(HERE), *targets], check=True)


def have_ref() -> bool:
    return REF_SO.exists()


class _Lib:
    def __init__(self, path: Path, prefix: str):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.lib = C.CDLL(str(path))
        self.prefix = prefix

    def fn(self, name, argtypes, restype=C.c_int):
        f = getattr(self.lib, self.prefix + name)
        f.argtypes = argtypes
        f.restype = restype
        return f


class Reference(_Lib):
    """ctypes view of the reference's own C++ API (oracle/_ref/libnnref.so)."""

    def __init__(self, path: Path = REF_SO):
        super().__init__(path, "nnref_")
        self._err = self.fn("last_error", [], C.c_char_p)

    def _check(self, st, idx=None):
        if st != 0:
            raise OracleError(st, self._err().decode(), idx)

    def worker_count(self) -> int:
        return self.fn("worker_count", [], C.c_uint)()

    def gaussian(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n)
        self.fn("gaussian", [C.c_uint64, C.c_int64, _dp], None)(seed, n, _ptr(out))
        return out

    def random_spd(self, n: int, cond: float, seed: int) -> np.ndarray:
        out = np.empty((n, n), np.complex128)
        self._check(self.fn("random_spd", [C.c_int64, C.c_double, C.c_uint64, _dp])(n, cond, seed, _ptr(out)))
        return out

    def direct_inverse(self, m):
        """nn::direct_inverse_oracle; OracleError(11, ..., pivot) on SingularMatrixError."""
        m = _z(m)
        out = np.empty_like(m)
        piv = C.c_int(-1)
        st = self.fn("direct_inverse_z", [_dp, C.c_int64, _dp, _ip])(_ptr(m), m.shape[0], _ptr(out), C.byref(piv))
        if st == 11:
            raise OracleError(st, self._err().decode(), piv.value)
        self._check(st)
        return out

    def random_conditioned_complex(self, n: int, cond: float, seed: int) -> np.ndarray:
        out = np.empty((n, n), np.complex128)
        f = self.fn("random_conditioned_complex", [C.c_int64, C.c_double, C.c_uint64, _dp])
        self._check(f(n, cond, seed, _ptr(out)))
        return out

    def random_sparse_spd(self, n: int, density: float, seed: int):
        f = self.fn("random_sparse_spd", [C.c_int64, C.c_double, C.c_uint64, _i64p, _dp, _dp, _dp])
        nnz = C.c_int64()
        self._check(f(n, density, seed, C.byref(nnz), None, None, None))
        rp, col, val = np.empty(n + 1, np.int64), np.empty(nnz.value, np.int64), np.empty(nnz.value)
        self._check(f(n, density, seed, C.byref(nnz), _ptr(rp), _ptr(col), _ptr(val)))
        return rp, col, val

    def matmul(self, a, b):
        a, b = _z(a), _z(b)
        out = np.empty((a.shape[0], b.shape[1]), np.complex128)
        n3 = C.c_double()
        f = self.fn("matmul_z", [_dp, _dp, C.c_int64, C.c_int64, C.c_int64, _dp, _dp])
        self._check(f(_ptr(a), _ptr(b), a.shape[0], a.shape[1], b.shape[1], _ptr(out), C.byref(n3)))
        return out, n3.value

    def residual_eps(self, x, a) -> float:
        x, a = _z(x), _z(a)
        eps = C.c_double()
        self._check(self.fn("residual_eps_z", [_dp, _dp, C.c_int64, _dp])(_ptr(x), _ptr(a), a.shape[0], C.byref(eps)))
        return eps.value

    def frobenius(self, m) -> float:
        m = _z(m)
        out = C.c_double()
        r, c = m.shape
        self._check(self.fn("frobenius_z", [_dp, C.c_int64, C.c_int64, _dp])(_ptr(m), r, c, C.byref(out)))
        return out.value

    def trace(self, m) -> complex:
        m = _z(m)
        out = np.empty(2)
        self._check(self.fn("trace_z", [_dp, C.c_int64, _dp])(_ptr(m), m.shape[0], _ptr(out)))
        return complex(out[0], out[1])

    def elementwise(self, op: str, a, b=None, s: complex = 0):
        codes = {"add": 0, "sub": 1, "scale": 2, "identity_minus": 3, "plus_identity": 4}
        a = _z(a)
        b = _z(b) if b is not None else a
        out = np.empty_like(a)
        n2 = C.c_int64()
        f = self.fn("elementwise_z", [C.c_int, _dp, _dp, C.c_int64, C.c_int64, C.c_double, C.c_double, _dp, _i64p])
        self._check(f(codes[op], _ptr(a), _ptr(b), a.shape[0], a.shape[1], complex(s).real, complex(s).imag,
                      _ptr(out), C.byref(n2)))
        return out, n2.value

    def step(self, kind: str, x, a, depth: int = 1):
        which = {"nn": 0, "newton": 1, "chebyshev": 2}[kind]
        x, a = _z(x), _z(a)
        out = np.empty_like(x)
        n3 = C.c_double()
        f = self.fn("step_z", [C.c_int, _dp, _dp, C.c_int64, C.c_int64, _dp, _dp])
        self._check(f(which, _ptr(x), _ptr(a), a.shape[0], depth, _ptr(out), C.byref(n3)))
        return out, n3.value

    def ns_sum(self, x0, a, order: int):
        x0, a = _z(x0), _z(a)
        out = np.empty_like(a)
        n3 = C.c_double()
        f = self.fn("ns_sum_z", [_dp, _dp, C.c_int64, C.c_int64, _dp, _dp])
        self._check(f(_ptr(x0), _ptr(a), a.shape[0], order, _ptr(out), C.byref(n3)))
        return out, n3.value

    def chain(self, a, x0, p: int, max_iters: int, tol: float = 0.0):
        """SURVEY §8(c) explicit-X0 chain. Returns (X, eps_hist, iters, seconds)."""
        a, x0 = _z(a), _z(x0)
        n = a.shape[0]
        out = np.empty_like(a)
        hist = np.zeros(max_iters + 1)
        iters, fail, secs = C.c_int(), C.c_int(-1), C.c_double()
        f = self.fn("chain_z", [_dp, C.c_int64, _dp, C.c_int, C.c_int, C.c_double, _dp, _dp, _ip, _ip, _dp])
        st = f(_ptr(a), n, _ptr(x0), p, max_iters, tol, _ptr(out), _ptr(hist), C.byref(iters), C.byref(fail),
               C.byref(secs))
        self._check(st, fail.value)
        return out, hist[: iters.value + 1], iters.value, secs.value

    def nn_invert(self, w, theta: float, valid: bool, depth: int, max_nests: int, tol: float):
        w = _z(w)
        n = w.shape[0]
        out = np.empty_like(w)
        hist = np.zeros(max_nests + 2)
        hl, sr, alpha, fail = C.c_int64(), C.c_int(), C.c_double(), C.c_int(-1)
        counts = np.zeros(2)
        f = self.fn("nn_invert_z", [_dp, C.c_int64, C.c_double, C.c_int, C.c_int64, C.c_int64, C.c_double, _dp, _dp,
                                    _i64p, _dp, _ip, _dp, _ip])
        st = f(_ptr(w), n, theta, int(valid), depth, max_nests, tol, _ptr(out), _ptr(hist), C.byref(hl),
               _ptr(counts), C.byref(sr), C.byref(alpha), C.byref(fail))
        self._check(st, fail.value)
        return out, dict(history=hist[: hl.value].copy(), n3=counts[0], n2=int(counts[1]),
                         stopped="tolerance" if sr.value == 0 else "max_nests",
                         alpha=None if alpha.value < 0 else alpha.value)

    def solve_normal(self, a, b, depth: int, max_nests: int, tol: float):
        """nn::solve_normal_equations; raises OracleError(20) on NonConvergenceError."""
        a, b = _z(a), _z(b)
        n, k = a.shape[0], b.shape[1]
        x = np.empty((n, k), np.complex128)
        hist = np.zeros(max_nests + 2)
        hl, sr, bw, fail = C.c_int64(), C.c_int(), C.c_double(), C.c_int(-1)
        counts = np.zeros(2)
        f = self.fn("solve_normal_z", [_dp, C.c_int64, _dp, C.c_int64, C.c_int64, C.c_int64, C.c_double, _dp, _dp,
                                       _i64p, _dp, _ip, _dp, _ip])
        st = f(_ptr(a), n, _ptr(b), k, depth, max_nests, tol, _ptr(x), _ptr(hist), C.byref(hl), _ptr(counts),
               C.byref(sr), C.byref(bw), C.byref(fail))
        rep = dict(history=hist[: hl.value].copy(), n3=counts[0], n2=int(counts[1]),
                   stopped="tolerance" if sr.value == 0 else "max_nests")
        if st == 20:
            raise OracleError(st, "NonConvergenceError", rep)
        self._check(st, fail.value)
        return x, rep, bw.value

    def theta_trace(self, w):
        w = _z(w)
        th, con, va = C.c_double(), C.c_double(), C.c_int()
        f = self.fn("theta_trace_z", [_dp, C.c_int64, _dp, _dp, _ip])
        self._check(f(_ptr(w), w.shape[0], C.byref(th), C.byref(con), C.byref(va)))
        return th.value, con.value, bool(va.value)

    def batched(self, mode: str, a, p: int, iters: int, threads: int = 1):
        """mode 'nn' (Jacobi X0, `iters` nests of depth p) or 'ns' (ns_sum of order `iters`)."""
        a = _z(a)
        b, n, _ = a.shape
        out = np.empty_like(a)
        eps = np.zeros(b)
        secs = C.c_double()
        f = self.fn("batched_z", [C.c_int, _dp, C.c_int64, C.c_int64, C.c_int, C.c_int, _dp, _dp, C.c_int, _dp])
        self._check(f(0 if mode == "nn" else 1, _ptr(a), b, n, p, iters, _ptr(out), _ptr(eps), threads,
                      C.byref(secs)))
        return out, eps, secs.value

    def spmv_block(self, row_ptr, col, val, x):
        row_ptr = np.ascontiguousarray(row_ptr, np.int64)
        col = np.ascontiguousarray(col, np.int32)
        val = np.ascontiguousarray(val, np.float64)
        x = _z(x)
        n = row_ptr.size - 1
        x2 = x.reshape(n, -1)
        out = np.empty_like(x2)
        f = self.fn("spmv_block", [_i64p, _i32p, _dp, C.c_int64, _dp, C.c_int64, _dp])
        self._check(f(_ptr(row_ptr, _i64p), _ptr(col, _i32p), _ptr(val), n, _ptr(x2), x2.shape[1], _ptr(out)))
        return out.reshape(x.shape)

    def sparse_factorized(self, row_ptr, col, val, b, gamma: int, theta: float):
        row_ptr = np.ascontiguousarray(row_ptr, np.int64)
        col = np.ascontiguousarray(col, np.int32)
        val = np.ascontiguousarray(val, np.float64)
        b = _z(b)
        n = row_ptr.size - 1
        b2 = b.reshape(n, -1)
        out = np.empty_like(b2)
        counts, secs, fail = np.zeros(1), C.c_double(), C.c_int(-1)
        f = self.fn("sparse_factorized", [_i64p, _i32p, _dp, C.c_int64, _dp, C.c_int64, C.c_int64, C.c_double, _dp,
                                          _dp, _dp, _ip])
        st = f(_ptr(row_ptr, _i64p), _ptr(col, _i32p), _ptr(val), n, _ptr(b2), b2.shape[1], gamma, theta,
               _ptr(out), _ptr(counts), C.byref(secs), C.byref(fail))
        self._check(st, fail.value)
        return out.reshape(b.shape), int(counts[0]), secs.value

    def ns_factorized(self, phi0, w, gamma: int):
        phi0, w = _z(phi0), _z(w)
        out = np.empty_like(w)
        n3 = C.c_double()
        f = self.fn("ns_factorized_z", [_dp, _dp, C.c_int64, C.c_int64, _dp, _dp])
        self._check(f(_ptr(phi0), _ptr(w), w.shape[0], gamma, _ptr(out), C.byref(n3)))
        return out, n3.value

    def power_ladder(self, p, e: int):
        p = _z(p)
        out = np.empty_like(p)
        n3 = C.c_double()
        f = self.fn("power_ladder_z", [_dp, C.c_int64, C.c_uint64, _dp, _dp])
        self._check(f(_ptr(p), p.shape[0], e, _ptr(out), C.byref(n3)))
        return out, n3.value

    def nn_explicit(self, phi0, w, nests: int, depth: int):
        phi0, w = _z(phi0), _z(w)
        out = np.empty_like(w)
        n3 = C.c_double()
        f = self.fn("nn_explicit_z", [_dp, _dp, C.c_int64, C.c_int64, C.c_int64, _dp, _dp])
        self._check(f(_ptr(phi0), _ptr(w), w.shape[0], nests, depth, _ptr(out), C.byref(n3)))
        return out, n3.value

    def equivalent_ns_order(self, nests: int, depth: int) -> int:
        return self.fn("equivalent_ns_order", [C.c_int64, C.c_int64], C.c_uint64)(nests, depth)


class Port(_Lib):
    """ctypes view of the plain-C restatement (oracle/lib/libnn_oracle.so)."""

    def __init__(self, path: Path = PORT_SO):
        super().__init__(path, "nno_")

    @staticmethod
    def _check(st, idx=None):
        if st != 0:
            raise OracleError(st, "oracle port failure", idx)

    def set_threads(self, t: int) -> None:
        self.fn("set_threads", [C.c_int], None)(t)

    def gaussian(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n)
        self.fn("gaussian", [C.c_uint64, C.c_int64, _dp], None)(seed, n, _ptr(out))
        return out

    def random_spd(self, n: int, cond: float, seed: int) -> np.ndarray:
        """nn::random_spd restated (real, float64), bit-identical to the reference's."""
        out = np.empty((n, n))
        self._check(self.fn("random_spd", [C.c_int64, C.c_double, C.c_uint64, _dp])(n, cond, seed, _ptr(out)))
        return out

    def matmul(self, a, b):
        a, b = _z(a), _z(b)
        out = np.empty((a.shape[0], b.shape[1]), np.complex128)
        f = self.fn("matmul_z", [_dp, _dp, C.c_int64, C.c_int64, C.c_int64, _dp])
        self._check(f(_ptr(a), _ptr(b), a.shape[0], a.shape[1], b.shape[1], _ptr(out)))
        return out

    def residual_eps(self, x, a) -> float:
        x, a = _z(x), _z(a)
        eps = C.c_double()
        self._check(self.fn("residual_eps_z", [_dp, _dp, C.c_int64, _dp])(_ptr(x), _ptr(a), a.shape[0], C.byref(eps)))
        return eps.value

    def nn_step(self, x, a, depth: int):
        x, a = _z(x), _z(a)
        out = np.empty_like(x)
        self._check(self.fn("nn_step_z", [_dp, _dp, C.c_int64, C.c_int64, _dp])(_ptr(x), _ptr(a), a.shape[0], depth,
                                                                                _ptr(out)))
        return out

    def ns_sum(self, x0, a, order: int):
        x0, a = _z(x0), _z(a)
        out = np.empty_like(a)
        self._check(self.fn("ns_sum_z", [_dp, _dp, C.c_int64, C.c_int64, _dp])(_ptr(x0), _ptr(a), a.shape[0], order,
                                                                               _ptr(out)))
        return out

    def chain(self, a, x0, p: int, max_iters: int, tol: float = 0.0):
        a, x0 = _z(a), _z(x0)
        out = np.empty_like(a)
        hist = np.zeros(max_iters + 1)
        iters, fail = C.c_int(), C.c_int(-1)
        f = self.fn("chain_z", [_dp, C.c_int64, _dp, C.c_int, C.c_int, C.c_double, _dp, _dp, _ip, _ip])
        st = f(_ptr(a), a.shape[0], _ptr(x0), p, max_iters, tol, _ptr(out), _ptr(hist), C.byref(iters),
               C.byref(fail))
        self._check(st, fail.value)
        return out, hist[: iters.value + 1], iters.value

    def batched(self, mode: str, a, p: int, iters: int, threads: int = 1):
        a = _z(a)
        b, n, _ = a.shape
        out = np.empty_like(a)
        eps = np.zeros(b)
        f = self.fn("batched_z", [C.c_int, _dp, C.c_int64, C.c_int64, C.c_int, C.c_int, _dp, _dp, C.c_int])
        self._check(f(0 if mode == "nn" else 1, _ptr(a), b, n, p, iters, _ptr(out), _ptr(eps), threads))
        return out, eps

    def spmv_block(self, row_ptr, col, val, x):
        row_ptr = np.ascontiguousarray(row_ptr, np.int64)
        col = np.ascontiguousarray(col, np.int32)
        val = np.ascontiguousarray(val, np.float64)
        x = _z(x)
        n = row_ptr.size - 1
        x2 = x.reshape(n, -1)
        out = np.empty_like(x2)
        f = self.fn("spmv_block_z", [_i64p, _i32p, _dp, C.c_int64, _dp, C.c_int64, _dp])
        self._check(f(_ptr(row_ptr, _i64p), _ptr(col, _i32p), _ptr(val), n, _ptr(x2), x2.shape[1], _ptr(out)))
        return out.reshape(x.shape)

    def sparse_factorized(self, row_ptr, col, val, b, gamma: int, theta: float):
        row_ptr = np.ascontiguousarray(row_ptr, np.int64)
        col = np.ascontiguousarray(col, np.int32)
        val = np.ascontiguousarray(val, np.float64)
        b = _z(b)
        n = row_ptr.size - 1
        b2 = b.reshape(n, -1)
        out = np.empty_like(b2)
        cnt, fail = C.c_int64(), C.c_int(-1)
        f = self.fn("sparse_factorized_z", [_i64p, _i32p, _dp, C.c_int64, _dp, C.c_int64, C.c_int64, C.c_double,
                                            _dp, _i64p, _ip])
        st = f(_ptr(row_ptr, _i64p), _ptr(col, _i32p), _ptr(val), n, _ptr(b2), b2.shape[1], gamma, theta,
               _ptr(out), C.byref(cnt), C.byref(fail))
        self._check(st, fail.value)
        return out.reshape(b.shape), cnt.value
