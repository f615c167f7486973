#!/bin/bash
# Static SASS opcode mix per kernel of librdfft.so:  tools/sass_mix.sh <regex-on-mangled-name>
cuobjdump -sass "${2:-paper_2511_01385_b200/librdfft.so}" | awk -v pat="$1" '
/Function : /{name=$3; keep = (name ~ pat); next}
keep && /^[ \t]+\/\*[0-9a-f]+\*\/[ \t]/{ op=$2; if (op ~ /^@/) op=$3; sub(/\..*/,"",op); sub(/;$/,"",op); cnt[name" "op]++ }
END{for(k in cnt) print cnt[k], k}' | sort -k2,2 -k1,1nr
