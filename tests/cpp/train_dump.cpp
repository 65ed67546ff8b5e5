// Driver for the training parity test (tests/test_gpu_training.py): runs
// ufpgd::train (include/ufpgd/training.hpp) on two UFPD files from an
// UnfoldedNetwork::pgd_init start and prints the history and the trained
// parameters as one JSON object.
//   train_dump train.ufpd val.ufpd L lambda0 loss_kind lambda_cost batch lr epochs patience seed
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <string>

#include "ufpgd/dataset.hpp"
#include "ufpgd/training.hpp"

int main(int argc, char** argv) {
  if (argc != 12) {
    std::fprintf(stderr, "usage: %s train.ufpd val.ufpd L lambda0 loss_kind lambda_cost batch lr epochs patience seed\n",
                 argv[0]);
    return 2;
  }
  try {
    const ufpgd::Dataset tr = ufpgd::read_dataset(argv[1]), va = ufpgd::read_dataset(argv[2]);
    const ufpgd::SystemConfig sys = ufpgd::SystemConfig::uniform(tr.num_users, tr.num_antennas, 10.0);
    const ufpgd::UnfoldedNetwork net =
        ufpgd::UnfoldedNetwork::pgd_init(tr.num_users, tr.num_antennas, std::atoi(argv[3]), std::atof(argv[4]));
    ufpgd::TrainConfig tc;
    tc.loss_kind = std::atoi(argv[5]) ? ufpgd::LossKind::kSupervised : ufpgd::LossKind::kUnsupervised;
    tc.lambda_cost = std::atof(argv[6]);
    tc.batch_size = std::atoi(argv[7]);
    tc.learning_rate = std::atof(argv[8]);
    tc.max_epochs = std::atoi(argv[9]);
    tc.patience = std::atoi(argv[10]);
    tc.seed = std::strtoull(argv[11], nullptr, 10);
    if (std::getenv("UFPGD_TRAIN_WARMUP")) {  // exclude CUDA context / module load from train_seconds
      ufpgd::TrainConfig warm = tc;
      warm.max_epochs = 1;
      (void)ufpgd::train(net, tr, va, warm, sys);
    }
    const auto t0 = std::chrono::steady_clock::now();
    const ufpgd::TrainResult r = ufpgd::train(net, tr, va, tc, sys);
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::printf("{\"epochs\": [");
    for (std::size_t i = 0; i < r.history.epochs.size(); ++i) {
      const ufpgd::EpochRecord& e = r.history.epochs[i];
      std::printf("%s[%ld, %.17g, %.17g, %.17g, %.17g]", i ? ", " : "", e.epoch, e.train_loss, e.val_loss,
                  e.val_mean_pcg, e.val_mean_sum_rate);
    }
    std::printf("], \"train_seconds\": %.6f, \"best_epoch\": %ld, \"stopping_epoch\": %ld, \"params\": [", secs,
                r.history.best_epoch, r.history.stopping_epoch);
    for (std::size_t i = 0; i < r.network.layers.size(); ++i)
      std::printf("%s%.17g, %.17g", i ? ", " : "", r.network.layers[i].lambda_i, r.network.layers[i].eta_i);
    std::printf("]}\n");
  } catch (const std::exception& e) {
    std::fprintf(stderr, "train_dump: %s\n", e.what());
    return 1;
  }
  return 0;
}
