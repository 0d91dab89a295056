# usage: ab_epi.sh "EPI LB DEBUG" ... -- M...
vars=(); while [ $# -gt 0 ] && [ "$1" != "--" ]; do vars+=("$1"); shift; done; shift
for v in "${vars[@]}"; do set -- $v "$@"; e=$1; l=$2; d=$3; shift 3
  TBIK_TC_EPI=$e TBIK_TC_LB=$l TBIK_TC_DEBUG=$d timeout 300 python tools/ab_epi.py "$@" 2>&1 | grep -v Warn | sed "s/^/dbg=$d /"; done
