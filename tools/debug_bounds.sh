#!/bin/bash
# Device-side bounds checks in place of compute-sanitizer (not available on
# this GPU pool): build the library with -DFGBD_DEBUG_BOUNDS=1 and run the
# GPU test suite and a 1M frame through it.  A failed FGBD_DCHECK traps.
set -e
python -c "from paper_2401_09721_b200._build import build; build(defines=('FGBD_DEBUG_BOUNDS=1',), lib='tools/_lib_debug.so')"
FGBD_LIB_PATH=tools/_lib_debug.so python -m pytest tests -m gpu -q -x -p no:cacheprovider
FGBD_LIB_PATH=tools/_lib_debug.so python tools/profile_frame.py --frames 2
FGBD_LIB_PATH=tools/_lib_debug.so python tools/profile_frame.py --frames 2 --kind constant --order shuffle
FGBD_LIB_PATH=tools/_lib_debug.so python tools/sanitize_run.py 20000
