# compute-sanitizer over the round-2 kernels (3xFP16 split / strips / two-pass,
# CORR strip statistics + zeroed-G Gram, scatter, side-stream fork/join) at the
# smallest sizes that take those paths
O=gpurun_out/san2
mkdir -p $O
for spec in "SYRK 256,256" "SYR2K 256,320" "CORR 256,256" "COVAR 300,257" "CORR 256,3008" "2MM 1792,1792,1792,1792" "2MM 1792,1792,3008,1792" "3MM 1792,1792,1792,1792,1792"; do
  set -- $spec
  for tool in memcheck racecheck synccheck; do
    if [ "$tool" = racecheck ] && [ "$1" = 2MM -o "$1" = 3MM ]; then continue; fi
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/profile_kernels.py $1 $2 stage=2 1 \
        > $O/${tool}_$1_$2.log 2>&1
    echo "$tool $1 $2: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/${tool}_$1_$2.log | tail -1)" >> $O/summary.txt
  done
done
cat $O/summary.txt
