"""Dense exp(tau K) action for tiny FD operators (test helper; scipy-free)."""

import numpy as np


def dense_expm_action(mats, tau, u):
    import cgl_oracle as O
    k = O.kron_sum_dense(mats)
    return O.unvec(O.expm(k, tau) @ O.vec(u), u.shape)
