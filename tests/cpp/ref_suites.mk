# tests/cpp/ref_suites.mk -- compiles the REFERENCE's own unit suites,
# UNMODIFIED and read in place from $(REF)/tests (never copied), against this
# repo's drop-in headers (include/catsim/) and libltl_b200.so, with the
# doctest-compatible harness tests/cpp/shim/doctest.h (the reference's vendor/
# doctest is absent, proj/.gitignore:2).  Run from the repo root:
#
#     make -f tests/cpp/ref_suites.mk            # -> build/ref_suites/test_*
#
# The binaries are git-ignored build products; they travel to the GPU box with
# the gpurun snapshot (build/ is not gpurun-ignored), where
# tests/test_ref_suites.py runs them.  Without $(REF) (the GPU box) nothing is
# rebuilt.
REF ?= /root/reference/proj
OUT ?= build/ref_suites
CXX ?= g++
SUITES := grid layout rule fragment cat_engine reference snapshot bench cost_model
EXTRA := $(OUT)/acceptance
CXXFLAGS := -std=c++20 -O2 -Wall -Wextra -Itests/cpp/shim -Iinclude -I$(REF)/tests -pthread
LDFLAGS := -Lpaper_2406_17284_b200 -lltl_b200 -Wl,-rpath,'$$ORIGIN/../../paper_2406_17284_b200'
HDRS := $(wildcard include/catsim/*.hpp) include/ltl_b200.h tests/cpp/shim/doctest.h

ifneq ($(wildcard $(REF)/tests/test_grid.cpp),)
all: $(SUITES:%=$(OUT)/test_%) $(EXTRA)
$(OUT)/test_%: $(REF)/tests/test_%.cpp $(HDRS) paper_2406_17284_b200/libltl_b200.so
	@mkdir -p $(OUT)
	$(CXX) $(CXXFLAGS) $< -o $@ $(LDFLAGS)
$(OUT)/acceptance: $(REF)/tests/acceptance.cpp $(HDRS) paper_2406_17284_b200/libltl_b200.so
	@mkdir -p $(OUT)
	$(CXX) $(CXXFLAGS) $< -o $@ $(LDFLAGS)
else
all:
	@echo "reference tests not found under $(REF); using prebuilt $(OUT)/ if present"
endif
.PHONY: all
