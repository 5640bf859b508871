"""a3 over NVLS (ihs_allreduce_multimem, nvls.cu) on ONE GPU: a world-size-1
group's symmetric buffer bound to a multicast address -- the reduction over
one rank is the identity, so the buffer must come back bit-identical, also on repeated calls (the
signal pads are left zero for the next one).
Skipped when torch gives no multicast mapping on the box."""
import os

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def group():
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
    yield dist.group.WORLD
    if own:
        dist.destroy_process_group()


@pytest.mark.parametrize("count", [1, 1000, 1024 * 128 + 128, 4096 * 96 + 96])
def test_nvls_allreduce_world1(group, count):
    from paper_1910_14166_b200.dist import NvlsAllreduce
    dev = torch.device("cuda", 0)
    try:
        ar = NvlsAllreduce(count, dev, group=group)
    except Exception as e:  # noqa: BLE001
        pytest.skip(f"no multicast mapping: {type(e).__name__}: {e}")
    g = torch.Generator(device=dev).manual_seed(count)
    t = torch.randn(count, dtype=torch.float64, device=dev, generator=g)
    ref = t.clone()
    for _ in range(3):  # the pads must be reusable
        ar(t)
    torch.cuda.synchronize()
    assert torch.equal(t, ref)
