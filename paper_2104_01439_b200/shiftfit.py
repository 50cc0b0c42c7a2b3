"""Refit of the shift-exponent map sigma_p from shift-search records
(PAPER.md:446-451): minimise the weighted loss
    loss_p = sum_i w_{l_i}^-2 (sigma_hat_i - sigma_p(k_i, l_i))^2,  w_l = N_l / |D|,
over (k_c0, k_c1, alpha_0, alpha_1) with Adam (learning rate 1e-3, init
(0.1, 1.0, -0.5, 1.0), 50 000 epochs in the paper).  Host-side CPU work on the
records hh_shift_search produces; the map itself is evaluated on the device by
the library (hh_problem_desc.shift_map) for solves.
"""
from __future__ import annotations

import numpy as np
import torch


def sigma_map_torch(w, k, l):
    kc = w[1] * torch.exp(w[0] * l)
    alpha = w[3] * torch.exp(w[2] * l)
    b = 2.0 - torch.exp(-alpha * (k - kc))
    return torch.clamp(b, 1.0, 2.0)


def fit_sigma_map(k, l, sigma_hat, init=(0.1, 1.0, -0.5, 1.0), lr=1e-3, epochs=50_000):
    """Returns (coefficients (k_c0, k_c1, alpha_0, alpha_1), final loss)."""
    k = torch.as_tensor(np.asarray(k, dtype=np.float64))
    l = torch.as_tensor(np.asarray(l, dtype=np.float64))
    s = torch.as_tensor(np.asarray(sigma_hat, dtype=np.float64))
    ln = l.numpy()
    wl = torch.as_tensor(np.array([np.mean(ln == v) for v in ln]))
    w = torch.tensor(init, dtype=torch.float64, requires_grad=True)
    opt = torch.optim.Adam([w], lr=lr)
    for _ in range(epochs):
        opt.zero_grad()
        loss = torch.sum(wl ** -2 * (s - sigma_map_torch(w, k, l)) ** 2)
        loss.backward()
        opt.step()
    with torch.no_grad():
        final = float(torch.sum(wl ** -2 * (s - sigma_map_torch(w, k, l)) ** 2))
    return tuple(float(v) for v in w.detach()), final
