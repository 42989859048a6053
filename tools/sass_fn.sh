#!/bin/bash
# usage: tools/sass_fn.sh <mangled-name-substring> : SASS of one kernel of libclgen_b200.so (address + text)
LIB=${LIB:-/root/repo/paper_1406_1215_b200/libclgen_b200.so}
cuobjdump -sass "$LIB" | awk -v pat="$1" '
/Function : /{on = index($0, pat) > 0}
on && /^[ \t]+\/\*[0-9a-f]{4}\*\//{sub(/^[ \t]+\/\*/,""); sub(/\*\/[ \t]+/," "); sub(/\/\*.*/,""); print}'
