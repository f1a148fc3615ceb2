"""B200-native RxGS receiver-conditioned render path (arXiv 2605.24290).

The product is the native library ``librxgs_b200.so`` (C-ABI in
``include/rxgs_b200.h``, hand-written sm_100a kernels in ``csrc/``).  This
package only exposes a ctypes binding of that C-ABI (``capi``) for Python
callers; there is no Python compute path and no CPU fallback.
"""
__all__ = ["capi"]
