#!/bin/bash
# The GPU suite against the bounds-checked build (RLC_DEBUG_CHECKS): the
# pool's compute-sanitizer is closed, so device index checks of our own stand
# in for memcheck.  usage: tests/run_checked.sh [pytest args]
set -e
cd "$(dirname "$0")/.."
make -s -C paper_1911_10217_b200/csrc OUT=$PWD/ab/lib_checked.so OBJ=$PWD/build/obj_checked \
  EXTRA=-DRLC_DEBUG_CHECKS
RLC_LIB_PATH=$PWD/ab/lib_checked.so python -m pytest tests -m gpu -q "$@"
