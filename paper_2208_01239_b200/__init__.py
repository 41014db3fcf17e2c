"""B200-native Frobenius inversion of complex matrices (arXiv 2208.01239).

The product is the C-ABI CUDA library ``libfrobinv.so`` (include/frobinv.h); this
package only builds it (``build.py``) and binds it (``frobinv.py``).
"""
from .frobinv import (  # noqa: F401
    FrobError, dev_status, dgemm, dgetrf, dinv, dpoinv, draw_mu, dtrmm, hpd_inv, inv, inv_batched, inv_batched_host,
    inv_dev, inv_host, inv_host_many, inv_rand, load, lyapunov, polar, sign, sylvester, zhpd_inv, zinv, zinv_batched,
)

__all__ = ["hpd_inv", "zhpd_inv", "sylvester", "lyapunov", "inv", "inv_dev", "dev_status", "inv_rand", "draw_mu",
           "inv_batched", "inv_host", "inv_host_many", "inv_batched_host", "zinv", "zinv_batched", "sign", "polar",
           "dgemm", "dtrmm", "dpoinv", "dinv", "dgetrf", "load", "FrobError"]
