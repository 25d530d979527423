"""pifcm-b200: the data-parallel hot path of 3DPIFCM (arXiv 2002.01981) on
B200 (sm_100a).  The product is libpifcm.so (C ABI, include/pifcm.h); this
package is its thin Python binding (argument marshalling only).
"""
from .api import (Context, IfcmConfig, PifcmError, PsoConfig, from_aos, pitch_of,  # noqa: F401
                  to_aos, to_pitched_x)

__version__ = "0.1.0"
