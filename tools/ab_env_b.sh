#!/bin/bash
# like ab_env.sh, on the variant-B library (paper_2007_04457_b200/lib_ab)
export HGR_B200_LIB=$(pwd)/paper_2007_04457_b200/lib_ab/libhgr_b200.so
exec bash $(dirname $0)/ab_env.sh "$@"
