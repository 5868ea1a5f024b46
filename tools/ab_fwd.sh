# A/B of two library builds on the same box, interleaved: bash tools/ab_fwd.sh A.so B.so [model rows ctx]
M=${3:-qwen3-14b}; R=${4:-1}; C=${5:-300}
for i in 1 2 3; do
  for L in "$1" "$2"; do echo -n "$(basename $L) "; DBL_LIB=$PWD/$L timeout 300 python tools/fwd_probe.py $M $R $C 30; done
done
