"""Host/device plumbing: every compute path runs on CUDA complex128 tensors.

Inputs may be numpy arrays (copied to the device, results copied back) or
torch CUDA tensors (stay on the device).  There is no CPU execution path.
"""

import numpy as np
import torch

from . import _lib


def to_device(x):
    """-> (C-contiguous complex128 CUDA tensor, came_from_host)."""
    _lib.require_cuda()
    if isinstance(x, torch.Tensor):
        if not x.is_cuda:
            return x.to(device="cuda", dtype=torch.complex128).contiguous(), True
        return x.to(dtype=torch.complex128).contiguous(), False
    a = np.ascontiguousarray(np.asarray(x, dtype=np.complex128))
    return torch.from_numpy(a).to("cuda", non_blocking=False), True


def to_host(t):
    """Device tensor -> numpy.  Fields of 1 MiB .. 4 GiB land in page-locked
    memory from torch's caching host allocator (a pageable .cpu() copy of a
    2 GiB state runs at a few GB/s; the pinned block is reused once the
    returned array is dropped); larger ones (1024^3: 17 GB) are not pinned."""
    nbytes = t.numel() * t.element_size()
    if nbytes < (1 << 20) or nbytes > (4 << 30):
        return t.cpu().numpy()
    try:
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    except RuntimeError:   # no page-locked memory to be had: pageable copy
        return t.cpu().numpy()
    h.copy_(t, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return h.numpy()


def to_host_if(t, host):
    return to_host(t) if host else t


def matrix_to_device(m):
    """Square/rectangular operator factor -> (M, M^T) contiguous on device."""
    if isinstance(m, torch.Tensor):
        d = m.to(device="cuda", dtype=torch.complex128)
    else:
        d = torch.from_numpy(np.ascontiguousarray(np.asarray(m, dtype=np.complex128))).cuda()
    return d.contiguous(), d.transpose(0, 1).contiguous()
