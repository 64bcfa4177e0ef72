#!/bin/bash
# spills.sh [pattern]: LDL/STL of one fused kernel instance with source lines (default: the bench's <8,256,0,1>)
PAT=${1:-fused_run_kernelILi8ELi256ELb0ELb1E}
D=$(mktemp -d); R=$(cd "$(dirname "$0")/.." && pwd); cd $D
cuobjdump -xelf all $R/paper_1805_11144_b200/build/fused.cu.o > /dev/null
nvdisasm -g *.cubin 2>/dev/null | awk -v pat="$PAT" '
  /^[ \t]*\.section[ \t]+\.text\./ { on = index($0, pat) > 0 }
  on && /\/\/## File/ { f = $0; sub(/.*kernels\//, "", f) }
  on && /(LDL|STL)/ { line = $0; gsub(/^[ \t]+/, "", line); print f " | " substr(line, 1, 70) }'
rm -rf $D
