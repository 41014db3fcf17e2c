"""B200-native Frobenius inversion of complex matrices (arXiv 2208.01239).

The product is the C-ABI CUDA library ``libfrobinv.so`` (include/frobinv.h); this
package only builds it (``build.py``) and binds it (``frobinv.py``).
"""
from .frobinv import (  # noqa: F401
    FrobError, dgemm, dgetrf, dinv, draw_mu, hpd_inv, inv, inv_batched, inv_host, inv_host_many, inv_batched_host, inv_rand, load, lyapunov, polar, sign, sylvester, zinv,
    zinv_batched, zhpd_inv,
)

__all__ = ["hpd_inv", "zhpd_inv", "sylvester", "lyapunov", "inv", "inv_rand", "draw_mu", "inv_batched", "inv_host", "inv_host_many", "inv_batched_host", "zinv", "zinv_batched", "sign", "polar", "dgemm", "dinv",
           "dgetrf", "load", "FrobError"]
