# ORACLE recipe (test infrastructure only): compile the reference simulator's own sources, where
# they lie under /root/reference, into oracle/_ref/libref_sim.a.  Used by tests/test_c5_replay_cpu.py
# to pin the config-5 harness's restatement of generate_trace / DualCache / tuner (tools/lb_sim.*)
# against the reference itself.  Never copied into the repo; outputs only under oracle/_ref/.
# nlohmann/json is not vendored by the reference (proj/vendor absent); the cudnn_frontend copy
# (3.11.3) in this image provides the header.
REF ?= /root/reference/proj
JSON ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty
OUT := _ref
SRCS := synth dual_cache tuner trace router sim
OBJS := $(addprefix $(OUT)/,$(addsuffix .o,$(SRCS)))

LBX := ../paper_2605_19385_b200

all: $(OUT)/libref_sim.a $(OUT)/ref_binding

# the reference-side binding (tools/ref_binding.cpp): reference simulator + this repo's C ABI
$(OUT)/ref_binding: ../tools/ref_binding.cpp $(OUT)/libref_sim.a $(LBX)/liblbx.so
	g++ -std=c++20 -O2 -I$(REF)/include -I../include $< $(OUT)/libref_sim.a -L$(LBX) -llbx \
	  -Wl,-rpath,'$$ORIGIN/../../paper_2605_19385_b200' -lpthread -o $@

$(OUT)/%.o: $(REF)/src/%.cpp
	@mkdir -p $(OUT)
	g++ -std=c++20 -O2 -fPIC -I$(REF)/include -I$(JSON) -c $< -o $@

$(OUT)/libref_sim.a: $(OBJS)
	ar rcs $@ $^

clean:
	rm -rf $(OUT)
.PHONY: all clean
