"""CPU-side checks of the C-ABI boundary: the library builds, loads and
exports every symbol include/mpwsd.h declares; without a GPU the decoder
refuses to run (no CPU fallback)."""
import ctypes

import pytest
import torch

from paper_2602_08501_b200 import _native


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    declared = _native.declared_symbols()
    assert "mpw_two_stage_batch" in declared and len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name


def test_abi_version():
    assert _native.lib().mpw_version() == 2


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU refusal")
def test_no_gpu_means_loud_failure():
    from paper_2602_08501_b200.decoders import DeviceDecoder
    from paper_2602_08501_b200 import configs
    with pytest.raises(_native.NativeError):
        DeviceDecoder(configs.CONFIGS["cfg1"].code())
    h = ctypes.c_void_p()
    assert _native.lib().mpw_create(0, ctypes.byref(h)) == -5   # MPW_ERR_NO_DEVICE
