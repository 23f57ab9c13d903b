"""PEC-sphere Mie series (test helper; the physics pin of the generator, §V.C.1).

Amplitude functions S1, S2 of Bohren & Huffman in the perfectly-conducting
limit: a_n = psi_n'(x)/xi_n'(x), b_n = psi_n(x)/xi_n(x), psi_n = x j_n,
xi_n = x h_n^(1). Bistatic RCS in the E-plane: sigma = lambda^2/pi |S2|^2 with
the scattering angle measured from the propagation direction. Truncation
n_max = ceil(x + 4 x^{1/3} + 2) (Wiscombe).
"""
import numpy as np
import scipy.special as sp


def mie_pec_S(ka: float, theta: np.ndarray):
    x = float(ka)
    nmax = int(np.ceil(x + 4 * x ** (1 / 3) + 2))
    n = np.arange(1, nmax + 1)
    jn = sp.spherical_jn(n, x)
    jnp = sp.spherical_jn(n, x, True)
    yn = sp.spherical_yn(n, x)
    ynp = sp.spherical_yn(n, x, True)
    psi, dpsi = x * jn, jn + x * jnp
    hn, dhn = jn + 1j * yn, jnp + 1j * ynp
    xi, dxi = x * hn, hn + x * dhn
    a, b = dpsi / dxi, psi / xi
    mu = np.cos(theta)
    S1 = np.zeros(mu.shape, complex)
    S2 = np.zeros(mu.shape, complex)
    pim1, pi = np.zeros_like(mu), np.ones_like(mu)
    for k in range(1, nmax + 1):
        if k > 1:
            pim1, pi = pi, ((2 * k - 1) / (k - 1)) * mu * pi - (k / (k - 1)) * pim1
        tau = k * mu * pi - (k + 1) * pim1
        c = (2 * k + 1) / (k * (k + 1))
        S1 += c * (a[k - 1] * pi + b[k - 1] * tau)
        S2 += c * (a[k - 1] * tau + b[k - 1] * pi)
    return S1, S2


def mie_eplane_rcs(ka: float, lam: float, scat_angle: np.ndarray) -> np.ndarray:
    _, S2 = mie_pec_S(ka, scat_angle)
    return lam ** 2 / np.pi * np.abs(S2) ** 2
