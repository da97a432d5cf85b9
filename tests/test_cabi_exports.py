"""CPU-only checks of the drop-in boundary: libvrg.so loads (no GPU needed to dlopen it) and
exports every symbol include/vrg.h declares; the ctypes table covers the header."""
import ctypes as C

from paper_1604_02153_b200 import _capi


def test_library_exports_header_symbols():
    lib = C.CDLL(_capi.LIB_PATH)
    missing = [s for s in _capi.header_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_ctypes_table_matches_header():
    assert sorted(_capi._SIG) == _capi.header_symbols()


def test_load_sets_signatures():
    lib = _capi.load()
    assert lib.vrg_version().decode().startswith("vrg")


def test_no_gpu_errors_are_reported():
    """Without a usable device the context call fails with a status, not a crash."""
    import torch

    lib = _capi.load()
    h = C.c_void_p()
    code = lib.vrg_ctx_create(0, None, C.byref(h))
    if torch.cuda.is_available():
        assert code == 0
        lib.vrg_ctx_destroy(h)
    else:
        assert code == _capi.VRG_RUNTIME_ERROR
        assert lib.vrg_last_error(None)
