# Fixed cost of one sspd CLI process on a B200 box: a bare CUDA process (tools/bin/cuinit from tools/cuinit.cu,
# built by tools/Makefile) vs sspd detect on a 300-record trace.  Run through gpurun.
nvidia-smi -q | grep -i "persistence" 
B=paper_1803_11036_b200/bin/sspd
W=$(mktemp -d)
printf 'slots 1\nbackground hosts=10 zipf=1.1 pairs-per-slot=300 max-distinct=4\n' > $W/tiny
$B synth $W/tiny --seed 1 -o $W/tiny.bin
for rep in 1 2 3 4; do
  s=$(date +%s%N); ./tools/bin/cuinit; e=$(date +%s%N); echo "bare CUDA process: $(( (e - s) / 1000000 )) ms"
  s=$(date +%s%N); $B detect $W/tiny.bin -o /dev/null; e=$(date +%s%N); echo "sspd detect tiny: $(( (e - s) / 1000000 )) ms"
done
