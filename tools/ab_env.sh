# A/B step timing over an environment variable (run under gpurun):
#   bash tools/ab_env.sh <tag> VAR v1 v2 ...
T=$1; V=$2; shift 2; O=gpurun_out/$T; mkdir -p $O
for rep in 1 2; do
  for x in "$@"; do
    echo "== $V=$x rep $rep" >> $O/ab.txt
    env $V=$x timeout 200 python tools/step_probe.py time >> $O/ab.txt 2>&1
  done
done
cat $O/ab.txt
