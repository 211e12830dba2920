#!/bin/bash
# time every exp/*.so variant with tools/sweep.py (W=8 lines); experiments only
for f in exp/*.so; do echo "== $f"; MRV_LIB_PATH=$f python tools/sweep.py ${1:-cfg5} ${2:-262144} 2>&1 | grep "W= 8"; done
