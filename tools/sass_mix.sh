#!/bin/bash
# instruction mix of one kernel's SASS: tools/sass_mix.sh <lib.so> <mangled name>
cuobjdump -sass -fun "$2" "$1" | grep -oE "^\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?[A-Z0-9_]+(\.[A-Z0-9_]+)*" | awk '{print $NF}' | sed 's/\..*//' | sort | uniq -c | sort -rn | awk '{s+=$1; printf "%s:%s ", $2, $1} END {print " total", s}'
