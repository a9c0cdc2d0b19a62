#!/bin/bash
# Opcode histogram of one kernel's SASS: tools/sass_hist.sh <lib.so> <mangled-name-substring>
cuobjdump -sass "$1" | awk -v pat="$2" '/Function : /{on = index($0, pat) > 0} on' |
  grep -oE "^\s+/\*[0-9a-f]+\*/\s+[A-Z0-9._]+" | awk '{print $2}' | sort | uniq -c | sort -rn
