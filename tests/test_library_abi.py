"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/mnl.h declares, and
rejects bad arguments before touching a device (no compute calls here: there is no GPU)."""
import ctypes
import os
import re

import pytest

import paper_1404_3177_b200 as M
from paper_1404_3177_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mnl.h")


@pytest.fixture(scope="module")
def lib():
    B.build()
    return M.load()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mnl_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for n in ("mnl_eval", "mnl_newton_fit", "mnl_num_params", "mnl_status_string"):
        assert n in names


def test_every_declared_symbol_is_exported(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr)
    assert set(M.EXPORTED) <= set(declared_functions())


def test_num_params_and_status_strings(lib):
    assert M.num_params(4, 1, 1, 1) == 11          # Fish model
    assert M.num_params(100, 49) == 4950           # Table 1 problem X
    assert M.num_params(100, 50) == 5049           # c4
    assert M.num_params(50, 30, 10, 5) == 1779     # c5
    assert M.num_params(1, 3) == -1
    assert M.status_string(0) == "MNL_OK"
    assert M.status_string(3) == "MNL_ERR_NOT_SPD"
    assert M.status_string(6) == "MNL_MAXITER"
    assert M.status_string(99) == "MNL_UNKNOWN"


def test_argument_errors_are_reported_without_a_device(lib):
    fake = ctypes.c_void_p(1 << 20)  # never dereferenced: validation fails first
    # K < 2
    assert lib.mnl_eval(10, 1, 2, 0, 0, fake, None, None, fake, fake, fake, None, None, None) == M.MNL_ERR_ARG
    # negative sizes / too large
    assert lib.mnl_eval(10, 4, -1, 0, 0, fake, None, None, fake, fake, fake, None, None, None) == M.MNL_ERR_ARG
    assert lib.mnl_eval(10, 300, 2, 0, 0, fake, None, None, fake, fake, fake, None, None, None) == M.MNL_ERR_ARG
    # N < 1
    assert lib.mnl_eval(0, 4, 2, 0, 0, fake, None, None, fake, fake, fake, None, None, None) == M.MNL_ERR_ARG
    # X required iff p > 0; Y iff f > 0; Z iff d > 0
    assert lib.mnl_eval(10, 4, 2, 0, 0, None, None, None, fake, fake, fake, None, None, None) == M.MNL_ERR_ARG
    assert lib.mnl_eval(10, 4, 0, 1, 0, None, None, None, fake, fake, fake, None, None, None) == M.MNL_ERR_ARG
    assert lib.mnl_eval(10, 4, 0, 0, 1, None, None, None, fake, fake, fake, None, None, None) == M.MNL_ERR_ARG
    # misaligned pointer
    bad = ctypes.c_void_p((1 << 20) + 8)
    assert lib.mnl_eval(10, 4, 2, 0, 0, bad, None, None, fake, fake, fake, None, None, None) == M.MNL_ERR_ARG
    it, ll = ctypes.c_int32(), ctypes.c_double()
    # tol <= 0, max_iter < 0
    assert lib.mnl_newton_fit(10, 4, 2, 0, 0, fake, None, None, fake, None, 0.0, 5, fake, ctypes.byref(it),
                              ctypes.byref(ll), None) == M.MNL_ERR_ARG
    assert lib.mnl_newton_fit(10, 4, 2, 0, 0, fake, None, None, fake, None, 1e-6, -1, fake, ctypes.byref(it),
                              ctypes.byref(ll), None) == M.MNL_ERR_ARG
    assert lib.mnl_eval_host(10, 1, 2, 0, 0, fake, None, None, fake, fake, fake, None, None) == M.MNL_ERR_ARG
    assert lib.mnl_cholesky(0, fake, None) == M.MNL_ERR_ARG
    # the later entry points validate the same way before touching a device
    assert lib.mnl_hessvec(10, 4, 2, 0, 0, fake, None, None, fake, fake, fake, fake, None) == M.MNL_ERR_ARG  # v == hv
    assert lib.mnl_std_errors(10, 1, 2, 0, 0, fake, None, None, fake, fake, fake, None) == M.MNL_ERR_ARG
    assert lib.mnl_std_errors(10, 4, 2, 0, 0, fake, None, None, fake, fake, None, None) == M.MNL_ERR_ARG  # se
    assert lib.mnl_predict(0, 4, 2, 0, 0, fake, None, None, fake, fake, None) == M.MNL_ERR_ARG
    assert lib.mnl_predict(10, 4, 2, 0, 0, fake, None, None, fake, bad, None) == M.MNL_ERR_ARG  # misaligned P
    assert lib.mnl_eval_async(10, 4, 2, 0, 0, fake, None, None, fake, fake, fake, None, None, None,
                              None) == M.MNL_ERR_ARG  # status pointer required
    assert lib.mnl_sym_pack(0, fake, fake, None) == M.MNL_ERR_ARG
    # shape queries: the BASELINE configs are supported; p = 255 with K = 256 exceeds the pass-1 bound
    for N, K, p, f, d in [(1000, 4, 3, 2, 1), (20000, 10, 20, 0, 0), (100000, 20, 50, 0, 0),
                          (500000, 100, 50, 0, 0), (200000, 50, 30, 10, 5)]:
        assert lib.mnl_check_shape(N, K, p, f, d) == M.MNL_OK
    assert lib.mnl_check_shape(15, 129, 7, 4, 8) == M.MNL_OK      # gradient partials in global scratch
    assert lib.mnl_check_shape(10, 256, 255, 0, 0) == M.MNL_ERR_ARG  # beyond the p bound for K > 128
    assert lib.mnl_check_shape(10, 256, 31, 0, 0) == M.MNL_OK
    assert lib.mnl_check_shape(10, 32, 127, 0, 0) == M.MNL_OK and lib.mnl_check_shape(10, 32, 128, 0, 0) == M.MNL_ERR_ARG
    assert lib.mnl_check_shape(10, 4, 2, 0, 65) == M.MNL_ERR_ARG
    assert lib.mnl_check_shape(10, 1, 2, 0, 0) == M.MNL_ERR_ARG
    assert lib.mnl_sym_unpack(5, None, fake, None) == M.MNL_ERR_ARG
    opts = M.FitOptions(0.0, 0.0, 5, 0, 0, 0.0)  # gtol <= 0
    assert lib.mnl_newton_fit_opts(10, 4, 2, 0, 0, fake, None, None, fake, None, ctypes.byref(opts), fake,
                                   ctypes.byref(it), ctypes.byref(ll), None, None) == M.MNL_ERR_ARG
    # the data-parallel fit: an all-reduce callback is required; options are validated the same way
    good = M.FitOptions(1e-6, 0.0, 5, 0, 0, 0.0)
    noop = M.ALLREDUCE_FN(lambda buf, n, st, ctx: 0)
    assert lib.mnl_newton_fit_dp(10, 4, 2, 0, 0, fake, None, None, fake, None, ctypes.byref(good),
                                 M.ALLREDUCE_FN(), None, fake, ctypes.byref(it), ctypes.byref(ll), None,
                                 None) == M.MNL_ERR_ARG
    assert lib.mnl_newton_fit_dp(10, 4, 2, 0, 0, fake, None, None, fake, None, ctypes.byref(opts), noop, None,
                                 fake, ctypes.byref(it), ctypes.byref(ll), None, None) == M.MNL_ERR_ARG
    assert lib.mnl_newton_fit_dp(10, 1, 2, 0, 0, fake, None, None, fake, None, ctypes.byref(good), noop, None,
                                 fake, ctypes.byref(it), ctypes.byref(ll), None, None) == M.MNL_ERR_ARG


def test_check_shape_sweep_runs_every_pass1_planner(lib):
    """mnl_check_shape plans pass 1 on the host (k_eval.cu's paths, the team mapping, the two-group
    X-only kernel): a sweep over the shape space, with and without the planners' size thresholds,
    returns MNL_OK or MNL_ERR_ARG for every shape inside the documented limits (no crash, no hang)."""
    seen = set()
    for force in (False, True):
        for k in ("MNL_FORCE_YZW", "MNL_FORCE_XG"):
            if force:
                os.environ[k] = "1"
            else:
                os.environ.pop(k, None)
        try:
            for N in (1, 7, 8, 9, 4096, 8192, 200000):
                for K in (2, 3, 8, 9, 16, 17, 33, 50, 56, 57, 64, 65, 100, 128, 129, 256):
                    for p in (0, 1, 30, 31, 32, 33, 63, 64):
                        for f, d in ((0, 0), (2, 1), (10, 5), (16, 8), (3, 2), (18, 0), (0, 9)):
                            seen.add(lib.mnl_check_shape(N, K, p, f, d))
        finally:
            os.environ.pop("MNL_FORCE_YZW", None)
            os.environ.pop("MNL_FORCE_XG", None)
    assert seen <= {M.MNL_OK, M.MNL_ERR_ARG} and M.MNL_OK in seen


def test_library_is_sm100a_only():
    so = open(M.LIB_PATH, "rb").read()
    assert b"sm_100a" in so or b"compute_100a" in so


def test_product_path_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_1404_3177_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, fn
