#!/bin/bash
# usage: tools/sass_of.sh <object> <kernel-name-regex>  -> SASS of the first matching kernel
obj=$1; pat=$2
name=$(cuobjdump -sass "$obj" | grep -o "Function : [^ ]*" | sed 's/Function : //' | grep -E "$pat" | head -1)
cuobjdump -sass -fun "$name" "$obj" | grep -E "^\s+/\*[0-9a-f]{4}\*/" | sed -E 's@^\s+/\*([0-9a-f]+)\*/\s+@\1 @; s@\s*/\*.*@@'
