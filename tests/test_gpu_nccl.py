"""The NCCL transport of the multi-GPU data path, run once on the one GPU of this pool: a ONE-rank
communicator drives every resolved NCCL entry point through comm.cpp's NcclTransport (grouped send/recv to self,
the four allreduce kinds, the peer-table exchange, the fence, init / user-rank / destroy, and the symmetric-window
peer mapping of peer_map 1: ncclMemAlloc, ncclCommWindowRegister, the device-side ncclGetPeerPointer, whose address
must alias the buffer), results checked in the library (include/amr_debug.h amr_debug_nccl_selftest).  Two ranks cannot share one GPU under NCCL, so the
multi-rank exchanges themselves are covered by the loopback and multi-process transports (test_gpu_multirank.py,
test_gpu_multiproc.py)."""
import ctypes as C

import pytest

pytestmark = pytest.mark.gpu


def test_nccl_transport_selftest_one_rank():
    import torch  # noqa: F401  (loads torch's libnccl.so.2 for the library's dlopen)
    import paper_2508_05020_b200 as amr
    L = amr.load()
    L.amr_debug_nccl_selftest.argtypes = [C.c_void_p, C.c_char_p, C.c_int32]
    uid = C.create_string_buffer(amr.nccl_unique_id(), 128)
    msg = C.create_string_buffer(512)
    rc = L.amr_debug_nccl_selftest(C.cast(uid, C.c_void_p), msg, 512)
    assert rc == 0, (rc, msg.value.decode())
    assert msg.value.decode().startswith("ok")
    # peer_map 1: ncclMemAlloc + ncclCommWindowRegister + ncclGetPeerPointer (device) map the buffer
    assert "window ok" in msg.value.decode(), msg.value.decode()

    # peer_map 1 fence (NEXT #3): ncclDevCommCreate with one LSA barrier, and the stage fence as an
    # ncclLsaBarrierSession kernel (three fences issued and completed on the stream)
    assert "lsa barrier fence ok" in msg.value.decode(), msg.value.decode()
