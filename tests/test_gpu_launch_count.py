"""pf_last_launch_count (bench.py's gpu_launches) against CUPTI.

Every launch site in the library bumps a per-thread counter; a run reports
its delta (graph replays report the count recorded at capture). Here the
kernels CUPTI sees during one run (torch.profiler, CUDA activity) must
number exactly what the library reports, with and without CUDA graphs, and
for the skinny-patch configuration that adds split-K reduction launches.
"""
import numpy as np
import pytest
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2405_14430_b200 as pf

pytestmark = pytest.mark.gpu


def _cupti_kernels(fn):
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    return sum(1 for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
               and "Memcpy" not in e.name and "Memset" not in e.name)


@pytest.mark.parametrize("graphs", [False, True])
@pytest.mark.parametrize("L,hs,heads,p,N,M", [(4, 128, 4, 256, 2, 4), (2, 1152, 16, 4096, 1, 8)])
def test_reported_launches_match_cupti(graphs, L, hs, heads, p, N, M):
    S, W = 3, 1
    x0 = pf.make_initial_latent(0, p, hs)
    with pf.ToyDiTCuda(0, L, hs, heads, 4.0, p, N) as m:
        m.set_graphs(graphs)
        x = torch.from_numpy(x0.astype(np.float32)).cuda()
        st = torch.cuda.Stream()
        m.run_pipefusion_device(x.data_ptr(), S, M, W, 0.1, st.cuda_stream)  # capture / warm
        m.synchronize(st.cuda_stream)

        def one():
            m.run_pipefusion_device(x.data_ptr(), S, M, W, 0.1, st.cuda_stream)
            m.synchronize(st.cuda_stream)

        seen = _cupti_kernels(one)
        reported = m.last_launch_count()
    assert reported > 0
    assert seen == reported, (seen, reported)
