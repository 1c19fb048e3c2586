// capi_layer.cpp — extern "C" surface of libfsmoe.so (include/fsmoe_layer.h).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <exception>
#include <memory>
#include <string>

#include "ep_group.hpp"
#include "fsmoe/moe_layer.hpp"
#include "fsmoe_cuda.h"
#include "fsmoe_layer.h"

struct fsmoe_ep {
  fsmoe::EpGroup* g;
};
struct fsmoe_layer {
  fsmoe::MoELayer* l;
};

namespace {

thread_local std::string g_err;

}  // namespace

namespace fsmoe {
void set_layer_error(const std::string& msg) { g_err = msg; }
}  // namespace fsmoe

namespace {

template <class F>
int guard(F&& f) {
  try {
    f();
    return FSMOE_OK;
  } catch (const fsmoe::ConfigError& e) {
    g_err = e.what();
    return FSMOE_CONFIG_ERROR;
  } catch (const fsmoe::FitQualityError& e) {
    g_err = e.what();
    return 3;
  } catch (const fsmoe::InvariantError& e) {
    g_err = e.what();
    return FSMOE_INVARIANT_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return FSMOE_CUDA_ERROR;
  }
}

}  // namespace

extern "C" {

const char* fsmoe_layer_last_error(void) { return g_err.c_str(); }

int fsmoe_ep_unique_id(unsigned char out[128]) {
  return guard([&] {
    ncclUniqueId id;
    fsmoe::nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out, &id, 128);
  });
}

int fsmoe_ep_create(int world, int rank, const unsigned char id[128], int device, int max_ctas,
                    fsmoe_ep** out) {
  return guard([&] {
    if (world < 1 || rank < 0 || rank >= world) throw fsmoe::ConfigError("ep: bad world/rank");
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    *out = new fsmoe_ep{new fsmoe::EpGroup(world, rank, uid, device, max_ctas)};
  });
}

int fsmoe_ep_create_local(int world, int device, fsmoe_ep** out) {
  return guard([&] {
    if (world < 1 || world > FSMOE_MAX_PEERS) throw fsmoe::ConfigError("ep: world must be in [1, 8]");
    auto hub = std::make_shared<fsmoe::LocalHub>(world);
    for (int r = 0; r < world; ++r) out[r] = nullptr;
    try {
      for (int r = 0; r < world; ++r) out[r] = new fsmoe_ep{new fsmoe::EpGroup(hub, r, device)};
    } catch (...) {
      for (int r = 0; r < world; ++r)
        if (out[r]) {
          delete out[r]->g;
          delete out[r];
          out[r] = nullptr;
        }
      throw;
    }
  });
}

int fsmoe_ep_allreduce(fsmoe_ep* ep, void* buf, long long n, int f64, void* stream) {
  return guard([&] {
    if (!ep || (n > 0 && !buf)) throw fsmoe::ConfigError("ep allreduce: null group or buffer");
    if (n <= 0) return;
    fsmoe::throw_cuda(cudaSetDevice(ep->g->device()), "cudaSetDevice");
    ep->g->allreduce_sum(buf, static_cast<size_t>(n), f64 != 0, static_cast<cudaStream_t>(stream));
  });
}

int fsmoe_ep_destroy(fsmoe_ep* ep) {
  return guard([&] {
    if (ep) {
      delete ep->g;
      delete ep;
    }
  });
}

int fsmoe_layer_create(const fsmoe_layer_config* c, fsmoe_ep* ep, fsmoe_layer** out) {
  return guard([&] {
    if (!c) throw fsmoe::ConfigError("layer: null config");
    fsmoe::MoELayerConfig cfg;
    cfg.tokens = c->tokens;
    cfg.model_dim = c->model_dim;
    cfg.ffn_dim = c->ffn_dim;
    cfg.experts = c->experts;
    cfg.top_k = c->top_k;
    if (c->gate_kind < 0 || c->gate_kind > 3) throw fsmoe::ConfigError("gate: unknown gate kind");
    cfg.gate = static_cast<fsmoe::GateKind>(c->gate_kind);
    cfg.ffn = c->ffn_kind ? fsmoe::LayerConfig::Ffn::gated3 : fsmoe::LayerConfig::Ffn::simple;
    cfg.capacity = c->capacity;
    cfg.capacity_factor = c->capacity_factor > 0.0 ? c->capacity_factor : 1.0;
    cfg.unlimited_capacity = c->unlimited != 0;
    cfg.transport = c->transport;
    cfg.proj_dim = c->proj_dim;
    cfg.seed = c->seed;
    cfg.precision = c->precision ? fsmoe::Precision::f32 : fsmoe::Precision::bf16;
    cfg.r_fwd = c->r_fwd;
    cfg.r_bwd = c->r_bwd;
    cfg.device = c->device;
    cfg.dense_grad_elems = c->dense_grad_elems;
    for (int i = 0; i < c->n_ar_slices; ++i) cfg.ar_slices.push_back(c->ar_slices[i]);
    *out = new fsmoe_layer{new fsmoe::MoELayer(cfg, ep ? ep->g : nullptr)};
  });
}

int fsmoe_layer_destroy(fsmoe_layer* layer) {
  return guard([&] {
    if (layer) {
      delete layer->l;
      delete layer;
    }
  });
}

int fsmoe_layer_bind(fsmoe_layer* layer, const fsmoe_layer_params* p) {
  return guard([&] {
    fsmoe::MoEParams q;
    q.w_gate = p->w_gate;
    q.w_noise = p->w_noise;
    q.proj = p->proj;
    q.w1 = p->w1;
    q.w2 = p->w2;
    q.g_gate = p->g_gate;
    q.g_noise = p->g_noise;
    q.g_proj = p->g_proj;
    q.g_w1 = p->g_w1;
    q.g_w2 = p->g_w2;
    q.dense_grad = p->dense_grad;
    layer->l->bind(q);
  });
}

long long fsmoe_layer_capacity(const fsmoe_layer* layer) { return layer->l->capacity(); }

int fsmoe_layer_forward(fsmoe_layer* layer, const void* x, void* y, void* stream) {
  return guard([&] { layer->l->forward(x, y, stream); });
}

int fsmoe_layer_backward(fsmoe_layer* layer, const void* dy, void* dx, void* stream) {
  return guard([&] { layer->l->backward(dy, dx, stream); });
}

int fsmoe_layer_set_trace(fsmoe_layer* layer, int on) {
  return guard([&] { layer->l->set_trace(on != 0); });
}

long long fsmoe_layer_trace(const fsmoe_layer* layer, char* buf, long long cap) {
  std::string j = layer->l->trace_json();
  if (buf && cap > 0) {
    const size_t n = std::min<size_t>(j.size(), static_cast<size_t>(cap - 1));
    std::memcpy(buf, j.data(), n);
    buf[n] = '\0';
  }
  return static_cast<long long>(j.size()) + 1;
}

int fsmoe_layer_buffer(const fsmoe_layer* layer, const char* name, void** ptr, long long* bytes) {
  return guard([&] { *ptr = layer->l->buffer(name, bytes); });
}

}  // extern "C"
