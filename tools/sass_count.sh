#!/bin/bash
# Static SASS opcode histogram of the first function whose mangled name matches $1.
# Usage: tools/sass_count.sh <regex> [lib] [top]
lib=${2:-paper_2303_03964_b200/libtfdp.so}
cuobjdump -sass "$lib" 2>/dev/null | awk -v pat="$1" '
  /Function :/ { if (f) exit; if ($0 ~ pat) f=1; next }
  f && /^[ \t]+\/\*[0-9a-f]+\*\// { op=$2; if (op ~ /^@/) op=$3; sub(/\..*/, "", op); sub(/;/, "", op); c[op]++; n++ }
  END { printf "%6d total\n", n; for (o in c) printf "%6d %s\n", c[o], o }' | sort -k1 -nr | head -${3:-14}
