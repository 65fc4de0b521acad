"""B200-native (sm_100a) RFDiffusion graph-field integrator (arXiv 2302.00942).

The product is the C-ABI library ``lib/librfd.so`` (``include/rfd.h``); this
package adds only its ctypes binding (:mod:`.rfd`) and build script
(:mod:`.build`).
"""

from .rfd import (Plan, RFDError, launch_count, load_library, profile_enable,  # noqa: F401
                  profile_read)
