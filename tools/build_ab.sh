#!/bin/bash
# build the current csrc tree as variant B into paper_2007_04457_b200/lib_ab (objects in
# build/ab); extra nvcc flags (e.g. -DHGR_LINES16=1) as arguments
set -e
cd $(dirname $0)/../paper_2007_04457_b200/csrc
rm -rf ../../build/ab
make -s OUT=../lib_ab OBJDIR=../../build/ab EXTRA="$*" ../lib_ab/libhgr_b200.so
