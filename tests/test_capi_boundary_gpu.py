"""The C-ABI's host-link and collective entry points (include/autohete.h), called exactly as a
foreign host would bind them (ctypes, plain pointers): ah_copy_h2d / ah_copy_d2h between pinned
host memory from ah_host_alloc and device memory on an ah_stream_create stream, and the NCCL
collectives on a 1-rank communicator (the only rank count one GPU allows: identity semantics,
in place and out of place)."""
import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_copy_h2d_d2h_roundtrip(cuda_device, native):
    from paper_2503_01890_b200 import _native as N
    L = N.lib()
    n = (64 << 20) + 3  # odd size, > 64 MiB
    hp, hq, st = C.c_void_p(), C.c_void_p(), C.c_void_p()
    N.check(L.ah_host_alloc(C.byref(hp), n), "host alloc")
    N.check(L.ah_host_alloc(C.byref(hq), n), "host alloc")
    N.check(L.ah_stream_create(C.byref(st), 0), "stream")
    src = np.ctypeslib.as_array((C.c_uint8 * n).from_address(hp.value))
    dst = np.ctypeslib.as_array((C.c_uint8 * n).from_address(hq.value))
    src[:] = np.random.default_rng(0).integers(0, 256, n, dtype=np.uint8)
    dst[:] = 0
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    N.check(L.ah_copy_h2d(dev.data_ptr(), hp, n, st), "h2d")
    N.check(L.ah_copy_d2h(hq, dev.data_ptr(), n, st), "d2h")
    torch.cuda.synchronize()
    N.check(L.ah_stream_destroy(st), "stream destroy")
    assert np.array_equal(src, dst)
    N.check(L.ah_host_free(hp), "free")
    N.check(L.ah_host_free(hq), "free")


def test_copy_rejects_bad_pointer(cuda_device, native):
    from paper_2503_01890_b200 import _native as N
    dev = torch.empty(16, dtype=torch.uint8, device="cuda")
    rc = N.lib().ah_copy_h2d(dev.data_ptr(), C.c_void_p(16), 1 << 40, None)  # 1 TiB from a bogus address
    assert rc == -2 and N.lib().ah_last_error()


def test_nccl_collectives_one_rank(cuda_device, native):
    from paper_2503_01890_b200 import _native as N
    L = N.lib()
    uid = N.dp_unique_id()
    comm = C.c_void_p()
    N.check(L.ah_nccl_comm_create((C.c_uint8 * 128).from_buffer_copy(uid), 1, 0, C.byref(comm)), "comm")
    s = torch.cuda.current_stream().cuda_stream
    n = 1_000_003
    g = torch.randn(n, device="cuda").bfloat16()
    out = torch.empty_like(g)
    N.check(L.ah_nccl_reduce_scatter_bf16(g.data_ptr(), out.data_ptr(), n, comm, s), "rs")
    assert torch.equal(out, g)
    w = g.clone()
    N.check(L.ah_nccl_reduce_scatter_bf16(w.data_ptr(), w.data_ptr(), n, comm, s), "rs in place")
    N.check(L.ah_nccl_all_gather_bf16(w.data_ptr(), w.data_ptr(), n, comm, s), "ag in place")
    ag = torch.empty_like(g)
    N.check(L.ah_nccl_all_gather_bf16(g.data_ptr(), ag.data_ptr(), n, comm, s), "ag")
    f = torch.randn(4097, device="cuda")
    f0 = f.clone()
    N.check(L.ah_nccl_all_reduce(f.data_ptr(), f.numel(), 0, comm, s), "ar f32")
    N.check(L.ah_nccl_all_reduce(g.data_ptr(), n, 1, comm, s), "ar bf16")
    torch.cuda.synchronize()
    assert torch.equal(w, ag) and torch.equal(ag, out) and torch.equal(f, f0)
    assert L.ah_nccl_all_reduce(f.data_ptr(), 1, 7, comm, s) == -1  # bad dtype
    N.check(L.ah_nccl_comm_destroy(comm), "destroy")
