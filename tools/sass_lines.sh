#!/bin/bash
# List source lines of a SASS opcode pattern in the fp64 hot kernel of a built lib (dev aid).
# usage: tools/sass_lines.sh lib.so 'DSETP.MAX|DSETP.MIN'
lib=$(realpath "$1"); d=$(mktemp -d); cd $d; cuobjdump -xelf all "$lib" >/dev/null 2>&1
nvdisasm --print-line-info csph_fused.sm_100a.cubin 2>/dev/null | awk '/^_ZN2ck46_GLOBAL__N__[0-9a-f_]*csph_fused_cu_[0-9a-f]*17fused_step_kernelIdLi128ELb1ELi8ELi3ELi3ELb0E.*:$/{f=1;next} /^\/\/----/{if(f)exit} f' > k.dis
awk -v pat="$2" '/\/\/## File/{match($0,/"[^"]*", line [0-9]+/); loc=substr($0,RSTART,RLENGTH); gsub(/.*\//,"",loc); next} $0 ~ pat {print loc}' k.dis | sort | uniq -c | sort -rn
echo "total: $(grep -cE "$2" k.dis) of $(grep -cE '^\s+/\*[0-9a-f]{4}\*/' k.dis)"
rm -rf $d
