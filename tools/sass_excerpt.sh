#!/bin/bash
# SASS evidence for the production kernel: instruction histogram, the packed-FP32 / async-copy
# / vector-reduction instruction forms, and the dC inner loop.
#   bash tools/sass_excerpt.sh > profiles/round2_drive_fast_kernel_sass.txt
FUN=_ZN4sgns17drive_fast_kernelILi5ELi3ELi6ELb1ELb0ELb0EEEvNS_8FastArgsE
LIB=$(dirname "$0")/../paper_1604_04661_b200/libsgns_b200.so
T=$(mktemp)
cuobjdump -sass -fun $FUN "$LIB" 2>/dev/null > $T
echo "# cuobjdump -sass -fun $FUN paper_1604_04661_b200/libsgns_b200.so"
echo "# (drive_fast_kernel<NS=5,NCH=3,K1R=6,EXACT_K,!FULL,!PAIR>: the bench's d=300, K=5 instantiation)"
echo "## opcode histogram (static instruction count)"
grep -oE "^\s+/\*[0-9a-f]+\*/\s+(@!?U?P[0-9T] )?[A-Z0-9_]+" $T | awk '{print $NF}' | sort | uniq -c | sort -rn | head -30
echo "## packed FP32, async copies, vector reductions (full forms)"
grep -oE "(FFMA2|FMUL2|FADD2|LDGSTS|REDG|LDG)[A-Za-z0-9_.]*" $T | sort | uniq -c
echo "## dC pass inner loop (input-outer: one staged row = LDS.128 x2 + LDS.64, its error row = LDS.128 + LDS.64, 30 FFMA2 with the error as broadcast .F32 operand)"
L=$(grep -n "LDS.128" $T | tail -4 | head -1 | cut -d: -f1)
sed -n "$((L-24)),$((L+48))p" $T | grep -v '^\s*/\* 0x' | sed 's@ */\* 0x[0-9a-f]* \*/@@' | grep -v '^\s*$'
rm -f $T
