run() { P=$1; shift; for c in "$@"; do if [ $c = default ]; then unset IRL_E2E_CHUNKS; else export IRL_E2E_CHUNKS=$c; fi; r=$(timeout 300 python profiles/e2e_parts.py --parts $P 2>&1 | grep '^{'); echo "$P $c $r"; done; }
run 8 default 3,21 4,20 2,4,18 3,5,16 default 3,21
run 4 default 6,18 5,19 1,5,18 default 6,18
run 2 default 10,14 1,3,8,12 default 10,14
run 1 default 13,11 default
