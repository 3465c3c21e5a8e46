#!/bin/bash
# build the product library; print errors and fail loudly (dev aid)
cd "$(dirname "$0")/.." && make -s -C paper_2007_04457_b200/csrc -j8 > /tmp/mk.log 2>&1
rc=$?; grep -v "spill\|^$" /tmp/mk.log | head -30; exit $rc
