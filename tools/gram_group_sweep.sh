for g in 8 16 32; do
  sed -i "s/^constexpr int GO_GROUP = .*/constexpr int GO_GROUP = $g;/" paper_2505_21404_b200/csrc/gram_oz.cuh
  python -c "from paper_2505_21404_b200 import _build; _build.build_library()" > /dev/null 2>&1
  echo "GO_GROUP $g"; python tools/gram_clock.py 0 0 2>&1 | tail -2
done
