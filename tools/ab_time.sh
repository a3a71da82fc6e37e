# A/B device timing of the in-tree library against build_var_a/libdbp_b200.so
# (a previous build), alternating runs on the same box.
# usage: bash tools/ab_time.sh reps cfg...
R=$1; shift
for c in "$@"; do for i in 1 2 3; do
  echo -n "A(new) "; python tools/t2_time.py $c $R | tail -1
  echo -n "B(old) "; DBP_LIB=build_var_a/libdbp_b200.so python tools/t2_time.py $c $R | tail -1
done; done
