#!/bin/bash
# build the current csrc tree as variant B into paper_2007_04457_b200/lib_ab (objects in build/ab)
set -e
cd $(dirname $0)/../paper_2007_04457_b200/csrc
make -s OUT=../lib_ab OBJDIR=../../build/ab ../lib_ab/libhgr_b200.so
