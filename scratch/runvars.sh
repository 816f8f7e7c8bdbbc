#!/bin/bash
# run scratch/levels.py for each built variant: runvars.sh v1 v2 ...
cp paper_1710_11593_b200/libfractime_b200.so /tmp/lib_orig.so
for v in "$@"; do
  cp scratch/var/$v/libfractime_b200.so paper_1710_11593_b200/libfractime_b200.so
  python scratch/levels.py --tag $v ${LEVELS_ARGS}
done
cp /tmp/lib_orig.so paper_1710_11593_b200/libfractime_b200.so
