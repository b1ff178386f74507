#!/bin/bash
# Two-level tags: compile-time variants on C5a (stage ms), then one ncu --set full capture.
tools/c5a_quick.sh t2_off PASGAL_BCC_TAGS2=0
for v in "$@"; do
  tools/c5a_quick.sh t2_$v PASGAL_BCC_TAGS2=1 PASGAL_BCC_LIB=paper_2404_17101_b200/lib/variants/lib_$v.so
done
