"""The C-ABI splitter all-gather (luda_nccl_init_all /
luda_allgather_splitters) on the one GPU of a test box: a single-device
communicator from ncclCommInitAll and one from a unique id, each gathering
a sample array (recv == send for one rank); the multi-rank path is the gloo
test in test_subcompact.py plus bench_c5 on multi-GPU nodes."""
import ctypes

import pytest

pytestmark = pytest.mark.gpu


def test_allgather_single_rank_communicators():
    import torch

    from paper_2004_03054_b200 import _native
    L = _native.lib(0)
    payload = bytes(range(256)) * 3
    send = torch.frombuffer(bytearray(payload), dtype=torch.uint8).cuda()
    s = torch.cuda.current_stream()
    comms = []
    arr = (ctypes.c_void_p * 1)()
    _native.check(L.luda_nccl_init_all(1, (ctypes.c_int * 1)(0), arr))
    comms.append(arr[0])
    uid = (ctypes.c_uint8 * 128)()
    _native.check(L.luda_nccl_unique_id(uid))
    h = ctypes.c_void_p()
    _native.check(L.luda_nccl_init_rank(1, 0, uid, ctypes.byref(h)))
    comms.append(h.value)
    for c in comms:
        recv = torch.zeros(len(payload), dtype=torch.uint8, device="cuda")
        _native.check(L.luda_allgather_splitters(c, send.data_ptr(), recv.data_ptr(), len(payload), s.cuda_stream))
        s.synchronize()
        assert bytes(recv.cpu().numpy().tobytes()) == payload
        _native.check(L.luda_nccl_destroy(c))
