#!/bin/bash
# static SASS mix of one kernel in a cubin: tools/sass_count.sh CUBIN FUNC_REGEX
cuobjdump -sass "$1" | awk -v re="$2" '/Function : /{f = ($0 ~ re)} f' | grep -E "^\s+/\*[0-9a-f]+\*/" | \
  sed -E 's/^\s+\/\*[0-9a-f]+\*\/\s+(@!?U?P[0-9T] )?//' | awk '{print $1}' | sed 's/\..*//' | sort | uniq -c | sort -rn | head -${3:-14} | tr '\n' ' '; echo
