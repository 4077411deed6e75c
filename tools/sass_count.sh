#!/bin/bash
# Static SASS size / opcode counts of the fp64 hot specialisation of the fused kernel
# (fused_step_kernel<double,128,HASW=1,8,3,3,GEN=0>) in one or more libcsph builds (dev aid).
for lib in "$@"; do
  cuobjdump -sass "$lib" | awk '/Function : .*fused_step_kernelIdLi128ELb1ELi8ELi3ELi3ELb0E/{f=1;next} /Function :/{f=0} f' > /tmp/_hot.sass
  n=$(grep -cE "^\s+/\*[0-9a-f]{4,}\*/" /tmp/_hot.sass)
  echo "$(basename $lib): $n instr; $(grep -oE '(FSEL|DFMA|DMUL|DADD|DSETP|IMAD|MUFU|LDS|BRA|VOTE)[A-Z0-9._]*' /tmp/_hot.sass | sed 's/\..*//' | sort | uniq -c | sort -rn | tr '\n' ' ')"
done
