#!/bin/bash
# run prof_kernels against an alternative build of libfdmd (tuning experiments)
cp paper_2502_05339_b200/libfdmd.so /tmp/libfdmd_main.so
cp "$1" paper_2502_05339_b200/libfdmd.so
shift
"$@"
cp /tmp/libfdmd_main.so paper_2502_05339_b200/libfdmd.so
