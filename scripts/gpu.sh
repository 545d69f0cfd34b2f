#!/bin/bash
# The one runner for gpurun calls (round 2; replaces round 1's one-off scripts).
#
#   gpurun -- 'bash scripts/gpu.sh TAG STEP [STEP ...]'
#
# Every output goes to gpurun_out/TAG/.  Steps run in order; a step's exit code
# is appended to gpurun_out/TAG/status.txt and never stops the later steps.
#   smoke                      __graft_entry__.smoke()
#   tests[:EXPR]               pytest -m gpu (optionally -k EXPR; "+" in EXPR stands for " or ")
#   bw                         the box's HBM copy bandwidth (scripts/bw_probe.py)
#   bench:NAME:ARGS            python bench.py ARGS (commas -> spaces) > NAME.json
#   ref:NAME:ARGS              python bench.py --impl reference ARGS > NAME.json
#   launches:NAME:ARGS         the bench command plain, then ncu's launch list of it
#   ncu:NAME:REGEX:SKIP:COUNT:ARGS  the bench command plain, then ncu --set full of
#                              COUNT launches of kernels matching REGEX after SKIP
#                              ("+" in REGEX stands for "|", which the shell would pipe)
#   py:NAME:SCRIPT:ARGS        python SCRIPT ARGS > NAME.log
#   env:VAR=VALUE / unenv:VAR  set / clear an environment variable for the later steps
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=$1; shift
O=gpurun_out/$TAG
mkdir -p "$O"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,temperature.gpu --format=csv > "$O/smi.csv" 2>&1
st() { echo "$1=$2" >> "$O/status.txt"; }
for step in "$@"; do
  IFS=':' read -r kind a1 a2 a3 a4 a5 <<< "$step"
  case $kind in
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$O/smoke.log" 2>&1; st smoke $? ;;
    tests) if [ -n "$a1" ]; then K=(-k "${a1//+/ or }"); else K=(); fi
           timeout 2400 python -m pytest tests -q -m gpu -rfE --durations=15 "${K[@]}" > "$O/pytest_gpu.log" 2>&1
           st tests $? ;;
    bw) timeout 120 python scripts/bw_probe.py > "$O/bw.json" 2>&1; st bw $? ;;
    bench) timeout 1200 python bench.py ${a2//,/ } > "$O/$a1.json" 2> "$O/$a1.err"; st "bench_$a1" $? ;;
    ref) timeout 900 python bench.py --impl reference ${a2//,/ } > "$O/$a1.json" 2> "$O/$a1.err"; st "ref_$a1" $? ;;
    launches) CMD="python bench.py ${a2//,/ }"
              timeout 900 $CMD > "$O/$a1.plain.log" 2>&1 && \
              timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
                  --log-file "$O/$a1.launches.csv" $CMD > "$O/$a1.ncu.log" 2>&1
              st "launches_$a1" $? ;;
    ncu) CMD="python bench.py ${a5//,/ }"
         timeout 900 $CMD > "$O/$a1.plain.log" 2>&1 && \
         timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:${a2//+/|}" -s "$a3" \
             -c "$a4" -o "$O/$a1" $CMD > "$O/$a1.ncu.log" 2>&1
         st "ncu_$a1" $? ;;
    env) export "$a1"; echo "env $a1" >> "$O/status.txt" ;;
    unenv) unset "$a1"; echo "unenv $a1" >> "$O/status.txt" ;;
    py) timeout 1200 python "$a2" ${a3//,/ } > "$O/$a1.log" 2>&1; st "py_$a1" $? ;;
    *) st "unknown_$step" 1 ;;
  esac
done
cat "$O/status.txt"
