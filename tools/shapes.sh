# solver-shape sweep (G K RPL) on the bench grids; usage: bash tools/shapes.sh [grids...]
GRIDS=${@:-"--grid 7:256 --grid 27:128 --grid 7:128"}
echo "auto"; timeout 300 python tools/devbench.py $GRIDS --ctas 148 --reps 10 --strategies 2 2>&1 | grep strategy
for sh in "1 4 2" "1 8 2" "2 4 2" "4 2 4" "4 4 4"; do set -- $sh; echo "G=$1 K=$2 rpl=$3"; HEC_WAVE_G=$1 HEC_WAVE_K=$2 HEC_WAVE_RPL=$3 timeout 300 python tools/devbench.py $GRIDS --ctas 148 --reps 10 --strategies 2 2>&1 | grep strategy; done
