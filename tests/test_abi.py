"""CPU checks of the drop-in boundary: the C-ABI libraries load and export every
symbol their headers declare (no compute calls: there is no GPU here)."""
import ctypes as C
import os
import re

import pytest

from paper_2103_08932_b200 import dev

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INC = os.path.join(ROOT, "include", "tlsph")
LIB = os.path.join(ROOT, "paper_2103_08932_b200", "lib")


def declared(header):
    text = open(os.path.join(INC, header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tlsph_[a-z0-9_]+)\s*\(", text)))


@pytest.mark.parametrize("header,lib", [("tlsph_dev.h", "libtlsph_cuda.so"), ("tlsph.h", "libtlsph.so.1")])
def test_every_declared_symbol_is_exported(header, lib):
    names = declared(header)
    assert len(names) >= 14
    L = C.CDLL(os.path.join(LIB, lib))
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_reference_c_abi_surface():
    # the 14 entry points of proj/include/tlsph/tlsph.h:31-68
    expected = {"tlsph_version", "tlsph_status_name", "tlsph_last_error", "tlsph_sim_create", "tlsph_sim_destroy",
                "tlsph_sim_run", "tlsph_sim_dim", "tlsph_sim_thread_count", "tlsph_sim_step_count",
                "tlsph_sim_damped_step_count", "tlsph_sim_phase_seconds", "tlsph_sim_probe_displacement",
                "tlsph_sim_settled", "tlsph_sim_settle_time"}
    assert set(declared("tlsph.h")) == expected


def test_c_abi_host_paths_without_gpu():
    L = C.CDLL(os.path.join(LIB, "libtlsph.so.1"))
    L.tlsph_version.restype = C.c_char_p
    L.tlsph_status_name.restype = C.c_char_p
    L.tlsph_last_error.restype = C.c_char_p
    L.tlsph_sim_phase_seconds.restype = C.c_double
    assert L.tlsph_version() == b"1.0.0"
    assert L.tlsph_status_name(0) == b"ok" and L.tlsph_status_name(2) == b"parse-error"
    # argument validation and config parsing run on the host (test_capi.cpp:81-97)
    assert L.tlsph_sim_create(None, None, 0, None) == 1
    sim = C.c_void_p()
    args = (C.c_char_p * 1)(b"case=unknown_case")
    assert L.tlsph_sim_create(None, args, 1, C.byref(sim)) == 2
    assert sim.value is None
    assert b"unknown case" in L.tlsph_last_error()
    args = (C.c_char_p * 2)(b"case=bending_cantilever", b"nonsense_key=1")
    assert L.tlsph_sim_create(None, args, 2, C.byref(sim)) == 2
    assert b"nonsense_key" in L.tlsph_last_error()
    # this build's extra key: GPU reduction mode
    args = (C.c_char_p * 2)(b"case=bending_cantilever", b"gpu.reduction=sideways")
    assert L.tlsph_sim_create(None, args, 2, C.byref(sim)) == 2
    assert b"gpu.reduction" in L.tlsph_last_error()
    args = (C.c_char_p * 2)(b"case=bending_cantilever", b"gpu.reduction=ordered")
    assert L.tlsph_sim_create(None, args, 2, C.byref(sim)) == 0
    L.tlsph_sim_destroy(sim)
    args = (C.c_char_p * 3)(b"case=bending_cantilever", b"resolution=6", b"threads=4")
    assert L.tlsph_sim_create(None, args, 3, C.byref(sim)) == 0
    assert L.tlsph_sim_dim(sim) == 3 and L.tlsph_sim_thread_count(sim) == 4
    assert L.tlsph_sim_step_count(sim) == 0
    assert L.tlsph_sim_phase_seconds(sim, b"total") < 0
    L.tlsph_sim_destroy(sim)
    L.tlsph_sim_destroy(None)
    assert L.tlsph_sim_run(None) == 1


def test_host_rng_matches_oracle():
    from oracle import oracle as O
    import numpy as np
    assert np.array_equal(dev.random_uniforms(7, 1000), O.random_uniforms(7, 1000))
    assert np.array_equal(dev.random_choice(26.5, 0.2, 0, 5000), O.random_choice(26.5, 0.2, 0, 5000))


def test_no_gpu_fails_loudly():
    if dev.device_count() > 0:
        pytest.skip("a GPU is present")
    import numpy as np
    with pytest.raises(dev.TlsphError) as e:
        dev.DeviceSystem(np.zeros((2, 2)) + [[0, 0], [0.1, 0]], 1.0, 1.0, 0.1)
    assert e.value.kind == "internal-error"


def test_device_abi_argument_validation_without_gpu():
    """The slab-linking and timing entry points validate their arguments on the host, exception-free
    (status codes, thread-local message), before touching a device."""
    L = C.CDLL(os.path.join(LIB, "libtlsph_cuda.so"))
    L.tlsph_dev_last_error.restype = C.c_char_p
    L.tlsph_dev_ipc_size.restype = C.c_size_t
    L.tlsph_dev_timer_stop.restype = C.c_double
    L.tlsph_dev_sweep_linked.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int]
    # IpcExport: header + 3 memory handles + 54 event handles (64 bytes each)
    assert L.tlsph_dev_ipc_size() >= 16 + 57 * 64
    assert L.tlsph_dev_sweep_linked(None, 0, 1, 1.0, 1e-4, 1) == 1
    assert b"no slabs" in L.tlsph_dev_last_error()
    arr = (C.c_void_p * 1)(None)
    assert L.tlsph_dev_sweep_linked(arr, 1, 1, 1.0, 1e-4, 1) == 1
    assert b"null slab" in L.tlsph_dev_last_error()
    assert L.tlsph_dev_sweep_linked(arr, 1, 0, 1.0, 1e-4, 1) == 1  # the explicit scheme is not swept
    assert L.tlsph_dev_ipc_export(None, None) == 1
    assert L.tlsph_dev_link_peer_ipc(None, 0, None, None) == 1
    assert L.tlsph_dev_timer_stop(None) < 0
