#!/bin/bash
# Static SASS op counts of the C4 temporal-blocking kernel (no GPU).
cd /tmp && nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -cubin -I/root/repo/include \
  -I/root/repo/paper_2307_07931_b200/csrc -Xptxas -v /root/repo/paper_2307_07931_b200/csrc/px_tb.cu -o /tmp/tb.cubin > /tmp/tb.log 2>&1 || { grep error /tmp/tb.log; exit 1; }
cuobjdump -res-usage /tmp/tb.cubin 2>&1 | grep -A1 "${1:-k_tbwILi0ELi4ELi1ELi0ELi0ELi1E}" | grep -o "REG:[0-9]*\|STACK:[0-9]*" | paste - -
cuobjdump -sass -fun "${2:-_ZN2px5k_tbwILi0ELi4ELi1ELi0ELi0ELi1EEEvNS_12StreamLaunchENS_8TbLaunchEiii}" /tmp/tb.cubin | grep -oE "^\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?[A-Z][A-Z0-9_.]*" | awk '{print $NF}' | sort | uniq -c | sort -rn | head -25
