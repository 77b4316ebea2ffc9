"""screen_sharded through NCCL (a process group of one on the one GPU of the
test box) against the oracle: the halo exchange is empty, everything else --
band planning, the band screen on the device, K5 over the band rows, the
NCCL all-gathers of counts and padded survivor rows, the device assembly --
runs as it does on 8 GPUs."""

import socket

import numpy as np
import pytest

import oracle as O
from conftest import packbits

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.fixture(scope="module")
def nccl_group(cuda):
    import torch.distributed as dist

    if dist.is_initialized():
        yield None
        return
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                            device_id=cuda)
    yield None
    dist.destroy_process_group()


@pytest.mark.parametrize("kw", [{}, {"alpha": 0.6, "beta": 1.6, "ladder_ratio": 1.2, "stride": 2}])
def test_screen_sharded_nccl_world1_vs_oracle(cuda, nccl_group, kw):
    import workloads as WL
    from paper_1707_05647_b200 import ScreeningConfig
    from paper_1707_05647_b200.sharding import screen_sharded

    img = WL.make_image(700, 520, seed=17, sigma=3.0, noise=1.0)
    case = WL.make_template(img, 18, 40, (0.8, 1.3), std_threshold=10.0)
    res = screen_sharded(img, case.template, ScreeningConfig(**kw), device=cuda)
    ref = O.screen(img, case.template, O.ScreeningConfig(**kw), nthreads=8)
    assert res.size_masks.rows == (0, img.shape[0])
    assert np.array_equal(res.candidates.array(), np.array(ref.candidates, np.int32).reshape(-1, 3))
    for m in ref.ladder:
        assert np.array_equal(packbits(res.size_masks[m]), packbits(ref.size_masks[m])), m
    assert np.array_equal(res.region_mask, ref.region_mask)
    assert (res.stats.patches_tested, res.stats.patches_kept, res.stats.region_pixels_kept) == \
        (ref.patches_tested, ref.patches_kept, ref.region_pixels_kept)
    # a second call reuses the cached band engine and the gather capacity
    res2 = screen_sharded(img, case.template, ScreeningConfig(**kw), device=cuda)
    assert res2.candidates == res.candidates
