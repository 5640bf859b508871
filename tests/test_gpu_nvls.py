"""a3 over NVLS (ihs_allreduce_multimem, nvls.cu) on ONE GPU.

One GPU per call on this pool, so the multi-rank sum cannot run here.  What
can: the kernel's whole path -- the signal-pad barrier, multimem.ld_reduce
.add.f64 on a multicast address and multimem.st -- on a multicast object of
ONE device, created here with the CUDA driver API (cuda-python; test plumbing
only, the arithmetic is the library's).  The sum over one rank is the
identity: the buffer must come back bit-identical, on repeated calls (the
protocol leaves the pads zero).  torch symmetric memory gives a world-size-1
group no multicast mapping, so that route (dist.NvlsAllreduce) is exercised
only when it does.  Skipped when the device has no multicast support."""
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ok(res, what=""):
    err = res[0] if isinstance(res, tuple) else res
    from cuda.bindings import driver as drv
    if err != drv.CUresult.CUDA_SUCCESS:
        raise RuntimeError(f"CUDA driver {what}: {err}")
    return res[1:] if isinstance(res, tuple) and len(res) > 2 else (res[1] if isinstance(res, tuple) and len(res) == 2 else None)


class SingleDeviceMulticast:
    """A physical allocation of `nbytes` on device 0 mapped at a unicast VA and
    bound to a one-device multicast object mapped at a multicast VA."""

    def __init__(self, nbytes: int):
        from cuda.bindings import driver as drv
        self.drv = drv
        torch.zeros(1, device="cuda:0")  # torch's primary context, current on this thread
        _ok(drv.cuInit(0), "init")
        dev = _ok(drv.cuDeviceGet(0), "device")
        mc_ok = _ok(drv.cuDeviceGetAttribute(drv.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev),
                    "attribute")
        if not mc_ok:
            raise RuntimeError("device has no multicast support")
        ht = drv.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
        mp = drv.CUmulticastObjectProp()
        mp.numDevices = 1
        mp.handleTypes = ht
        mp.size = max(nbytes, 1)
        gran = _ok(drv.cuMulticastGetGranularity(mp, drv.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED),
                   "granularity")
        ap = drv.CUmemAllocationProp()
        ap.type = drv.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        ap.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        ap.location.id = 0
        ap.requestedHandleTypes = ht
        agran = _ok(drv.cuMemGetAllocationGranularity(ap, drv.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_RECOMMENDED),
                    "alloc granularity")
        gran = max(int(gran), int(agran))
        size = (nbytes + gran - 1) // gran * gran
        mp.size = size
        self.size = size
        self.mc = _ok(drv.cuMulticastCreate(mp), "multicast create")
        _ok(drv.cuMulticastAddDevice(self.mc, dev), "add device")
        self.phys = _ok(drv.cuMemCreate(size, ap, 0), "mem create")
        _ok(drv.cuMulticastBindMem(self.mc, 0, self.phys, 0, size, 0), "bind")
        acc = drv.CUmemAccessDesc()
        acc.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = 0
        acc.flags = drv.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        self.uc_va = _ok(drv.cuMemAddressReserve(size, gran, 0, 0), "reserve uc")
        _ok(drv.cuMemMap(self.uc_va, size, 0, self.phys, 0), "map uc")
        _ok(drv.cuMemSetAccess(self.uc_va, size, [acc], 1), "access uc")
        self.mc_va = _ok(drv.cuMemAddressReserve(size, gran, 0, 0), "reserve mc")
        _ok(drv.cuMemMap(self.mc_va, size, 0, self.mc, 0), "map mc")
        _ok(drv.cuMemSetAccess(self.mc_va, size, [acc], 1), "access mc")

    def close(self):
        drv = self.drv
        drv.cuMemUnmap(self.mc_va, self.size)
        drv.cuMemUnmap(self.uc_va, self.size)
        drv.cuMemAddressFree(self.mc_va, self.size)
        drv.cuMemAddressFree(self.uc_va, self.size)
        drv.cuMulticastUnbind(self.mc, 0, 0, self.size)
        drv.cuMemRelease(self.phys)
        drv.cuMemRelease(self.mc)


@pytest.mark.parametrize("count", [1, 1000, 1024 * 128 + 128, 4096 * 96 + 96])
def test_nvls_allreduce_one_device(count):
    import paper_1910_14166_b200 as P
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    try:
        import cuda.bindings.driver  # noqa: F401
        mcb = SingleDeviceMulticast(count * 8)
    except Exception as e:  # noqa: BLE001
        pytest.skip(f"no single-device multicast object: {type(e).__name__}: {e}")
    try:
        dev = torch.device("cuda", 0)
        rng = np.random.default_rng(count)
        src = torch.from_numpy(rng.standard_normal(count)).to(dev)
        # the unicast view of the physical pages: fill and read back through copies
        drv = mcb.drv
        nb = count * 8
        torch.cuda.synchronize()
        _ok(drv.cuMemcpyDtoD(mcb.uc_va, src.data_ptr(), nb))
        pad = torch.zeros(1024, dtype=torch.int32, device=dev)
        pads = torch.tensor([pad.data_ptr()], dtype=torch.int64, device=dev)
        for _ in range(3):
            P.ihs_allreduce_multimem(int(mcb.mc_va), pads, 0, 1, count, pad.numel())
        torch.cuda.synchronize()
        out = torch.empty_like(src)
        _ok(drv.cuMemcpyDtoD(out.data_ptr(), mcb.uc_va, nb))
        torch.cuda.synchronize()
        assert torch.equal(out, src)
        assert int(pad.abs().sum()) == 0  # the barrier slots are left free
    finally:
        torch.cuda.synchronize()
        mcb.close()


def test_nvls_torch_symmetric_memory_world1():
    """The dist.NvlsAllreduce route (torch symmetric memory): runs only when
    torch gives the group a multicast mapping."""
    import torch.distributed as dist
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29547")
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        from paper_1910_14166_b200.dist import NvlsAllreduce
        try:
            ar = NvlsAllreduce(4096, dev)
        except Exception as e:  # noqa: BLE001
            pytest.skip(f"no multicast mapping from torch: {type(e).__name__}: {e}")
        t = torch.randn(4096, dtype=torch.float64, device=dev)
        ref = t.clone()
        ar(t)
        torch.cuda.synchronize()
        assert torch.equal(t, ref)
    finally:
        if own:
            dist.destroy_process_group()


def test_nvls_argument_errors():
    """ihs_allreduce_multimem's synchronous argument checks (nothing enqueued)."""
    import paper_1910_14166_b200 as P
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    dev = torch.device("cuda", 0)
    pads = torch.zeros(1, dtype=torch.int64, device=dev)
    buf = torch.zeros(16, dtype=torch.float64, device=dev)
    ctx = P.Context(0)
    L = P.lib()
    h = ctx._bind()
    import ctypes as C
    mc, pp = C.c_void_p(buf.data_ptr()), C.c_void_p(pads.data_ptr())
    assert L.ihs_allreduce_multimem(h, mc, pp, 1, 1, 16, 1024) == P.ERR_INVALID_ARGUMENT  # rank >= world
    assert L.ihs_allreduce_multimem(h, mc, pp, 0, 0, 16, 1024) == P.ERR_INVALID_ARGUMENT  # world < 1
    assert L.ihs_allreduce_multimem(h, mc, pp, 0, 1, -1, 1024) == P.ERR_INVALID_ARGUMENT  # count < 0
    assert L.ihs_allreduce_multimem(h, None, pp, 0, 1, 16, 1024) == P.ERR_INVALID_ARGUMENT  # no buffer
    assert L.ihs_allreduce_multimem(h, mc, pp, 0, 2, 1 << 24, 3) == P.ERR_UNSUPPORTED  # pads too small
    assert L.ihs_allreduce_multimem(h, mc, pp, 0, 1, 0, 0) == P.OK  # nothing to do
