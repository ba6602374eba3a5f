#!/bin/bash
# The GPU suite on the bounds-checked build (librpq_b200_checked.so): every
# device check must hold (a failure fails the run that hit it).
tag=${1:-checked}
out=gpurun_out
mkdir -p $out
RPQ_ENGINE=checked timeout -s KILL 2400 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $out/gpu_tests_checked_$tag.log 2>&1
echo "checked_tests_rc=$?"; tail -3 $out/gpu_tests_checked_$tag.log
