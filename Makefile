# Builds libsanta.so (the C-ABI product library) for B200 / sm_100a.
# The kernels are instantiated in one object per (launcher family, dtype, head_dim) from
# csrc/inst.cu so `make -j` compiles them in parallel; santa_abi.cu holds the C ABI.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           -Xptxas -v -Iinclude --expt-relaxed-constexpr
CSRC := paper_2605_01910_b200/csrc
HDR := $(wildcard $(CSRC)/*.cuh) include/santa.h
LIBDIR := paper_2605_01910_b200/_lib
OBJDIR := build/obj
LIB := $(LIBDIR)/libsanta.so

FAMS := Score Sample Prop Flash Step Dense Bern
DTS := bf16 f16 f32
DS := 64 128
T_bf16 := __nv_bfloat16
T_f16 := __half
T_f32 := float
INST_OBJS := $(foreach f,$(FAMS),$(foreach t,$(DTS),$(foreach d,$(DS),$(OBJDIR)/inst_$(f)_$(t)_$(d).o)))
OBJS := $(OBJDIR)/santa_abi.o $(OBJDIR)/peer_exchange.o $(INST_OBJS)

all: $(LIB)

$(OBJDIR)/santa_abi.o: $(CSRC)/santa_abi.cu $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $@.log || (cat $@.log; exit 1)

$(OBJDIR)/peer_exchange.o: $(CSRC)/peer_exchange.cu include/santa.h
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $@.log || (cat $@.log; exit 1)

# inst_<Fam>_<dtype>_<D>.o
$(OBJDIR)/inst_%.o: $(CSRC)/inst.cu $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $< -DSANTA_INST_FAM=Run$(word 1,$(subst _, ,$*)) \
	  -DSANTA_INST_T=$(T_$(word 2,$(subst _, ,$*))) -DSANTA_INST_D=$(word 3,$(subst _, ,$*)) 2> $@.log || (cat $@.log; exit 1)

$(LIB): $(OBJS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)
	@cat $(OBJDIR)/santa_abi.o.log $(OBJDIR)/peer_exchange.o.log $(INST_OBJS:=.log) > $(LIBDIR)/ptxas.log

sass: $(LIB)
	cuobjdump -sass $(LIB) > $(LIBDIR)/libsanta.sass

clean:
	rm -rf $(LIB) $(OBJDIR)

.PHONY: all clean sass
