#!/bin/bash
# Static SASS opcode counts of one kernel: tools/sass_count.sh LIB FUNC_SUBSTRING [N]
cuobjdump -sass "$1" | awk -v f="$2" '/Function :/{on = index($0, f) > 0} on' |
  grep -oE "^\s+/\*[0-9a-f]+\*/\s+[A-Z0-9_.]+" | awk '{print $2}' | sort | uniq -c | sort -rn | head -${3:-30}
