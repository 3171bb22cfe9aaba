"""Host control data (boxes, beam, path, local-box policy, macro schedule): re-exported
from the vendored copy of the reference's bookkeeping (``vendored/lpbfsim_control.py``)."""

from .vendored.lpbfsim_control import *  # noqa: F401,F403
from .vendored.lpbfsim_control import STEFAN_BOLTZMANN  # noqa: F401
