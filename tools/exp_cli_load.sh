# sspd detect on 4 router shard files: serial shard loading (tools/bin/sspd_serial, the CLI
# before concurrent loading, built by hand from git) vs the current CLI.  Run through gpurun:
#   /usr/local/graft/bin/gpurun -- 'bash tools/exp_cli_load.sh > gpurun_out/cli_load.txt 2>&1'
set -e
B=paper_1803_11036_b200/bin/sspd
W=$(mktemp -d)
printf 'slots 10\nbackground hosts=200000 zipf=1.1 pairs-per-slot=250000 max-distinct=16\nsuper cip=10.0.0.1 count=4096 from=0 to=9\n' > $W/spec
for i in 0 1 2 3; do
  $B synth $W/spec --seed 5ee$i -o $W/s$i.bin
  $B synth $W/spec --seed 5ee$i --format text -o $W/s$i.txt
done
ls -l $W
for fmt in bin text; do
  ext=$fmt; [ $fmt = text ] && ext=txt
  for impl in tools/bin/sspd_serial $B; do
    for rep in 1 2 3; do
      s=$(date +%s%N)
      $impl detect $W/s0.$ext $W/s1.$ext $W/s2.$ext $W/s3.$ext --format $fmt -o $W/out_$(basename $impl)_$fmt.csv
      e=$(date +%s%N)
      echo "$fmt $(basename $impl) run $rep: $(( (e - s) / 1000000 )) ms"
    done
  done
  cmp $W/out_sspd_serial_$fmt.csv $W/out_sspd_$fmt.csv && echo "$fmt: reports identical ($(wc -l < $W/out_sspd_$fmt.csv) rows)"
done
# in-process phases of one detect call (loading, then run_detection's own breakdown)
for fmt in bin text; do
  ext=$fmt; [ $fmt = text ] && ext=txt
  SSPD_PIPELINE_TIMING=1 $B detect $W/s0.$ext $W/s1.$ext $W/s2.$ext $W/s3.$ext --format $fmt -o /dev/null
done
# fixed cost of one detect call (CUDA init, grid lifetimes): a 1-slot, 300-record trace
printf 'slots 1\nbackground hosts=10 zipf=1.1 pairs-per-slot=300 max-distinct=4\n' > $W/tiny
$B synth $W/tiny --seed 1 -o $W/tiny.bin
for rep in 1 2 3; do
  s=$(date +%s%N); $B detect $W/tiny.bin -o /dev/null; e=$(date +%s%N)
  echo "tiny 1-shard trace run $rep: $(( (e - s) / 1000000 )) ms"
  s=$(date +%s%N); $B detect $W/tiny.bin $W/tiny.bin $W/tiny.bin $W/tiny.bin -o /dev/null; e=$(date +%s%N)
  echo "tiny 4-shard trace run $rep: $(( (e - s) / 1000000 )) ms"
done
rm -rf $W
