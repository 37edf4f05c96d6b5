"""On-device direct stencil summation (csrc/direct.cu)
against the MSBFM FFT path and the C oracle: both evaluate
FastForce::apply (convolution.hpp:249-259), so they must agree to round-off."""
import numpy as np
import pytest
import torch

from oracle.oracle import Oracle, Rng, random_field

M = 3


@pytest.mark.gpu
@pytest.mark.parametrize("dims", [(64, 64), (96, 40), (257, 130), (24, 24, 24), (20, 12, 17)])
def test_direct_matches_fft_and_oracle(dims):
    from paper_2301_11828_b200.engine import FastForce, build_kernel
    dim = len(dims)
    n = int(np.prod(dims))
    h = 1.0 / dims[0]
    K = build_kernel(dim, h, 3.015 * h, M, 1.0, 1.0 if dim == 2 else 0.0)
    ff = FastForce(dims, M, K)
    u_np = np.stack([random_field(Rng(5100 + i), dim, n) for i in range(2)])
    u = torch.from_numpy(u_np).cuda()
    f_fft = torch.empty_like(u)
    f_dir = torch.empty_like(u)
    st = torch.cuda.current_stream()
    ff.apply_device(u, f_fft, 2, stream=st)
    ff.apply_direct_device(u, f_dir, 2, stream=st)
    torch.cuda.synchronize()
    rel = float(torch.linalg.norm(f_dir - f_fft) / torch.linalg.norm(f_fft))
    assert rel <= 1e-12, rel
    o = Oracle(dims, h=h, delta=3.015 * h, M=M)
    o.set_kernel(K)
    ref = o.apply(u_np[0])
    got = f_dir[0].cpu().numpy()
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-12
    ff.close()
