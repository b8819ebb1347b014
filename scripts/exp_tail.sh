for t in "2,256" "1,512" "4,128" "8,64" "8,128"; do
  echo "== tail $t"; NSW_TAIL_TILE=$t python scripts/phase_timing.py | grep -A14 "tail launch" | grep "backward\|forward\|total\|Adam\|rebuild"
done
